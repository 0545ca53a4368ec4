#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "engines_agree or block_results or integer or ragged or full_size" > $OUT/pytest.log 2>&1
for R in 1 2 3 4 5; do
  timeout 300 python bench.py --engine 4 --R $R --B 1024 --steps 20 --warmup 5 --no-e2e --no-cpu --no-comparators > $OUT/engine4_R$R.json 2> $OUT/engine4_R$R.err
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:sp_async -s 2 -c 1 -o $OUT/async python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators --engine 4 > $OUT/ncu_async.log 2>&1
echo done > $OUT/DONE
