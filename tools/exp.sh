#!/bin/bash
# Quick GPU experiments: tcgen05 debug modes (0 normal, 1 TMA-only, 2 1-D bulk copies).
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
for m in 0 1 2; do
  TCR_DEBUG_MODE=$m timeout 300 python bench.py --engine 2 --steps 10 --warmup 3 --no-e2e --no-cpu --no-comparators > $OUT/tc05_mode$m.json 2> $OUT/tc05_mode$m.err
done
timeout 300 python bench.py --engine 1 --steps 10 --warmup 3 --no-e2e --no-cpu --no-comparators > $OUT/mma.json 2> $OUT/mma.err
echo done > $OUT/DONE
