OUT=gpurun_out/nat4; mkdir -p $OUT
L=LIB=build/ab/nat_fast_bt32.so
timeout 900 python tools/ab.py --n 268435456 --rounds 5 --reps 5 \
  m4r3_old:0:3:128:M=4,$L m4r3:0:3:128:M=4 m4r5_old:0:5:128:M=4,$L m4r5:0:5:128:M=4 m4r5b32_old:0:5:32:M=4,$L m4r5b32:0:5:32:M=4 \
  m2r3_old:0:3:128:M=2,$L m2r3:0:3:128:M=2 m4r6_old:0:6:1024:M=4,$L m4r6:0:6:1024:M=4 m4r32_old:0:32:128:M=4,$L m4r32:0:32:128:M=4 \
  m4r1:0:1:128:M=4 m4r1k:0:1:1024:M=4 m2r1:0:1:128:M=2 \
  > $OUT/ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fuzz" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x > $OUT/fuzz.log 2>&1; echo "exit $?" >> $OUT/fuzz.log
