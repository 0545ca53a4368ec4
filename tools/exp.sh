#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -rf -k "shuffle32 or half_tree or oracle64 or recurrence or split" > $OUT/pytest_var.log 2>&1
timeout 900 python -m pytest tests -m gpu -q > $OUT/pytest_all.log 2>&1
echo done > $OUT/DONE
