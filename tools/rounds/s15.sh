mkdir -p gpurun_out/s15
timeout 1200 python tools/ab.py --n 268435456 --rounds 9 --reps 10 u4n4:0:1:128:M=4,LIB=build_ab/lib_k1.so u2n8:0:1:128:M=4,LIB=build_ab/lib_u2n8.so u1n16:0:1:128:M=4,LIB=build_ab/lib_u1n16.so m16:0:1:128 > gpurun_out/s15/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 u4n4:0:1:128:M=4,LIB=build_ab/lib_k1.so u2n8:0:1:128:M=4,LIB=build_ab/lib_u2n8.so u1n16:0:1:128:M=4,LIB=build_ab/lib_u1n16.so > gpurun_out/s15/ab30.txt 2>&1
