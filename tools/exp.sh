#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
TCR_DEBUG_MODE=14 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "(block_results or integer or full_size or ordered) and not genm and not tcgen05 and not mma_sync-" > $OUT/pytest14.log 2>&1
timeout 1200 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_rot:4:1:1024:TCR_DEBUG_MODE=14 async_rot_d8:4:1:1024:TCR_DEBUG_MODE=14 async_R4B128:4:4:128 async_rot_R4B128:4:4:128:TCR_DEBUG_MODE=14 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
