#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
TCR_DEBUG_MODE=13 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "(engines_agree or block_results or integer or ragged or full_size or ordered or tree) and not genm" > $OUT/pytest13.log 2>&1
timeout 900 python tools/ab.py --out $OUT/ab.json async_cta:4:1:1024:TCR_DEBUG_MODE=12 async_stream:4:1:1024:TCR_DEBUG_MODE=13 async_stream_R2:4:2:1024:TCR_DEBUG_MODE=13 async_stream_R4B128:4:4:128:TCR_DEBUG_MODE=13 async_stream_R5B32:4:5:32:TCR_DEBUG_MODE=13 async_R4B128:4:4:128:TCR_DEBUG_MODE=12 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
