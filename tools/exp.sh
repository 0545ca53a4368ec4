#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x > $OUT/pytest_all.log 2>&1
timeout 1200 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_pf8:4:1:1024:TCR_DEBUG_MODE=8 async_contig:4:1:1024:TCR_DEBUG_MODE=15 async_g128k:4:1:1024:TCR_GROUP_TARGET=131072 async_R4B128:4:4:128 async_R2:4:2:1024 regs:3:1:1024 bulk:1:1:1024 tc05:2:1:1024 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
