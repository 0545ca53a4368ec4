mkdir -p gpurun_out/s14
timeout 1200 python tools/ab.py --n 268435456 --rounds 9 --reps 10 k1:0:1:128:M=4,LIB=build_ab/lib_k1.so k2:0:1:128:M=4 k1b64:0:1:64:M=4,LIB=build_ab/lib_k1.so k2b64:0:1:64:M=4 k1b1024:0:1:1024:M=4,LIB=build_ab/lib_k1.so k2b1024:0:1:1024:M=4 m16:0:1:128 > gpurun_out/s14/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 k1:0:1:128:M=4,LIB=build_ab/lib_k1.so k2:0:1:128:M=4 > gpurun_out/s14/ab30.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "m4 or genm or fuzz or from_single or natural or sides or overflow or ragged or edge" > gpurun_out/s14/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s14/pytest_gpu.log
