#!/bin/bash
# Quick GPU experiments: engines and profiling modes.
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "engines_agree or block_results or integer" > $OUT/pytest.log 2>&1
for e in 1 3; do
  timeout 300 python bench.py --engine $e --steps 10 --warmup 3 --no-e2e --no-cpu --no-comparators > $OUT/engine$e.json 2> $OUT/engine$e.err
done
TCR_DEBUG_MODE=1 timeout 300 python bench.py --engine 1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-comparators > $OUT/bulk_mode1.json 2> $OUT/bulk_mode1.err
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sp_bulk -s 2 -c 1 -o $OUT/bulk python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators --engine 1 > $OUT/ncu_bulk.log 2>&1
echo done > $OUT/DONE
