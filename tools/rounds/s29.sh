mkdir -p gpurun_out/s29
timeout 900 python tools/ab.py --n 268435456 --rounds 7 --reps 10 r3:0:3:128 r3d12:0:3:128:TCR_DEBUG_MODE=11 r5:0:5:128 r5d10:0:5:128:TCR_DEBUG_MODE=11 r3b1024:0:3:1024 r3b1024d12:0:3:1024:TCR_DEBUG_MODE=11 > gpurun_out/s29/ab28.txt 2>&1
timeout 900 python tools/ab.py --rounds 5 --reps 10 r3:0:3:128 r3d12:0:3:128:TCR_DEBUG_MODE=11 r5:0:5:128 r5d10:0:5:128:TCR_DEBUG_MODE=11 > gpurun_out/s29/ab30.txt 2>&1
