mkdir -p gpurun_out/s16
timeout 1200 python tools/ab.py --n 268435456 --rounds 9 --reps 10 u4n4:0:1:128:M=4,LIB=build_ab/lib_k1.so u8n2:0:1:128:M=4,LIB=build_ab/lib_u8n2.so > gpurun_out/s16/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 u4n4:0:1:128:M=4,LIB=build_ab/lib_k1.so u8n2:0:1:128:M=4,LIB=build_ab/lib_u8n2.so > gpurun_out/s16/ab30.txt 2>&1
