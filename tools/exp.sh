#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 300 python tools/dbg_bulk.py > $OUT/dbg.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q > $OUT/pytest_all.log 2>&1
echo done > $OUT/DONE
