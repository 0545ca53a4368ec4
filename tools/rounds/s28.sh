mkdir -p gpurun_out/s28
timeout 1200 python tools/ab.py --n 268435456 --rounds 7 --reps 10 r2old:0:2:128:M=4,LIB=build_ab/lib_r1only.so r2:0:2:128:M=4 r4old:0:4:128:M=4,LIB=build_ab/lib_r1only.so r4:0:4:128:M=4 r2b32old:0:2:32:M=4,LIB=build_ab/lib_r1only.so r2b32:0:2:32:M=4 r4b1024old:0:4:1024:M=4,LIB=build_ab/lib_r1only.so r4b1024:0:4:1024:M=4 > gpurun_out/s28/ab28.txt 2>&1
true
timeout 900 python -m pytest tests -m gpu -q -x -k "m4_register or fp32 or from_single or fuzz" > gpurun_out/s28/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s28/pytest.log
