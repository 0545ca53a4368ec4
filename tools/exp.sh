#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "block_results or integer or full_size or ordered or tree_and" > $OUT/pytest.log 2>&1
timeout 1200 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_g256k:4:1:1024:TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=262144 async_g128k:4:1:1024:TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=131072 async_g512k:4:1:1024:TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=524288 async_R4B128:4:4:128 async_R4B128_g256k:4:4:128:TCR_GROUP_CAP=1024,TCR_GROUP_TARGET=262144 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
