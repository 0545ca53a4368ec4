#!/bin/bash
OUT=gpurun_out/${1:-exp}
mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "engines_agree or block_results or integer or ragged or full_size or ordered or tree" > $OUT/pytest.log 2>&1
timeout 900 python tools/ab.py --out $OUT/ab.json async:4:1:1024 async_cta:4:1:1024:TCR_DEBUG_MODE=12 async_R2:4:2:1024 async_R2B128:4:2:128 async_R4B128:4:4:128 tc05:2:1:1024 tc05_2cta:2:1:1024:TCR_DEBUG_MODE=11 > $OUT/ab.txt 2>&1
echo done > $OUT/DONE
