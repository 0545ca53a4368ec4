mkdir -p gpurun_out/s25
timeout 900 python tools/ab.py --rounds 5 --reps 5 old:0:1:1024:FIN=ordered,LIB=build_ab/lib_pre_rec.so new:0:1:1024:FIN=ordered tree:0:1:1024 > gpurun_out/s25/u30.txt 2>&1
timeout 900 python tools/ab.py --n 268435456 --rounds 5 --reps 5 old:0:1:128:M=4,FIN=ordered,LIB=build_ab/lib_pre_rec.so new:0:1:128:M=4,FIN=ordered tree:0:1:128:M=4 old32:0:1:32:M=4,FIN=ordered,LIB=build_ab/lib_pre_rec.so new32:0:1:32:M=4,FIN=ordered > gpurun_out/s25/u28m4.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ordered or oracle64 or serial or chain or golden" > gpurun_out/s25/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s25/pytest.log
