#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1200 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_g32k:4:1:1024:TCR_GROUP_TARGET=32768 async_g128k:4:1:1024:TCR_GROUP_TARGET=131072 async_g256k:4:1:1024:TCR_GROUP_TARGET=262144 async_2cta:4:1:1024:TCR_CTAS_PER_SM=2 async_1cta:4:1:1024:TCR_CTAS_PER_SM=1 async_d8_4cta:4:1:1024:TCR_DEBUG_MODE=9,TCR_CTAS_PER_SM=4 async_d8_5cta:4:1:1024:TCR_DEBUG_MODE=9,TCR_CTAS_PER_SM=5 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
