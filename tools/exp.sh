#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -s -k "genm or default_config" > $OUT/pytest_genm.log 2>&1
timeout 900 python -m pytest tests -m gpu -q -x > $OUT/pytest_all.log 2>&1
echo done > $OUT/DONE
