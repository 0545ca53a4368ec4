#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_nopf:4:1:1024:TCR_DEBUG_MODE=8 bulk:1:1:1024 regs:3:1:1024 tc05:2:1:1024 async_R4B128:4:4:128 async_R5B32:4:5:32 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
