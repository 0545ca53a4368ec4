mkdir -p gpurun_out/s2
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/s2/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s2/pytest_gpu.log
timeout 900 python tools/ab.py --rounds 9 --reps 10 base:4:1:1024:LIB=build_ab/lib_base.so new:4:1:1024 t8:4:1:1024:TCR_TAIL_SPLIT=8 t8u4:4:1:1024:TCR_TAIL_SPLIT=8,TCR_TAIL_UNITS=4 t4u4:4:1:1024:TCR_TAIL_UNITS=4 t8u3:4:1:1024:TCR_TAIL_SPLIT=8,TCR_TAIL_UNITS=3 shuffle:0:1:1:SHUFFLE=1 probe:0:1:1:PROBE=1 > gpurun_out/s2/ab.txt 2>&1
timeout 600 python tools/ab.py --n 268435456 --rounds 7 --reps 10 base:4:1:1024:LIB=build_ab/lib_base.so new:4:1:1024 t8:4:1:1024:TCR_TAIL_SPLIT=8 baseR4:4:4:128:LIB=build_ab/lib_base.so newR4:4:4:128 shuffle:0:1:1:SHUFFLE=1 > gpurun_out/s2/ab28.txt 2>&1
timeout 300 python tools/timeline.py > gpurun_out/s2/timeline.txt 2>&1
