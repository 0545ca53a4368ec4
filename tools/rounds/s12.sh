mkdir -p gpurun_out/s12
timeout 1200 python tools/ab.py --n 268435456 --rounds 7 --reps 10 r3old:0:3:128:LIB=build_ab/lib_head.so r3:0:3:128 r5old:0:5:128:LIB=build_ab/lib_head.so r5:0:5:128 b512old:0:1:512:LIB=build_ab/lib_head.so b512:0:1:512 b96old:0:1:96:LIB=build_ab/lib_head.so b96:0:1:96 r3b1024old:0:3:1024:LIB=build_ab/lib_head.so r3b1024:0:3:1024 r1:0:1:128 shuffle:0:1:1:SHUFFLE=1 > gpurun_out/s12/ab28.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s12/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s12/pytest_gpu.log
