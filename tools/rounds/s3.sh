mkdir -p gpurun_out/s3
timeout 900 python tools/ab.py --rounds 9 --reps 10 base:4:1:1024:LIB=build_ab/lib_base.so new:4:1:1024 nopf:4:1:1024:TCR_DEBUG_MODE=21 shuffle:0:1:1:SHUFFLE=1 base2:4:1:1024:LIB=build_ab/lib_base.so new2:4:1:1024 nopf2:4:1:1024:TCR_DEBUG_MODE=21 > gpurun_out/s3/ab.txt 2>&1
