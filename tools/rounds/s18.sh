mkdir -p gpurun_out/s18
timeout 900 python tools/ab.py --rounds 5 --reps 5 old:0:1:1024:FIN=ordered,LIB=build_ab/lib_w512.so new:0:1:1024:FIN=ordered tree:0:1:1024 > gpurun_out/s18/u30.txt 2>&1
timeout 900 python tools/ab.py --rounds 5 --reps 5 --dist normal old:0:1:1024:FIN=ordered,LIB=build_ab/lib_w512.so new:0:1:1024:FIN=ordered tree:0:1:1024 > gpurun_out/s18/n30.txt 2>&1
timeout 900 python tools/ab.py --n 268435456 --rounds 5 --reps 5 old:0:1:128:M=4,FIN=ordered,LIB=build_ab/lib_w512.so new:0:1:128:M=4,FIN=ordered tree:0:1:128:M=4 > gpurun_out/s18/u28m4.txt 2>&1
timeout 900 python tools/ab.py --n 268435456 --rounds 3 --reps 2 --dist normal old:0:1:128:M=4,FIN=ordered,LIB=build_ab/lib_w512.so new:0:1:128:M=4,FIN=ordered tree:0:1:128:M=4 > gpurun_out/s18/n28m4.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ordered or ORDERED or serial or chain" > gpurun_out/s18/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s18/pytest.log
