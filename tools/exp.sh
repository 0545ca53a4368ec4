#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
TCR_DEBUG_MODE=15 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "(block_results or integer or full_size or ordered) and not genm" > $OUT/pytest15.log 2>&1
timeout 1200 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_g256k:4:1:1024:TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=262144 async_contig:4:1:1024:TCR_DEBUG_MODE=15 async_contig_g256k:4:1:1024:TCR_DEBUG_MODE=15,TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=262144 async_pf8:4:1:1024:TCR_DEBUG_MODE=8 async_contig_R4B128:4:4:128:TCR_DEBUG_MODE=15 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
