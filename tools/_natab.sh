OUT=gpurun_out/tr2; mkdir -p $OUT
L=LIB=build/ab/pre_tr.so
timeout 900 python tools/ab.py --n 268435456 --rounds 5 --reps 5 \
  m32r1_old:0:1:128:M=32,$L m32r1:0:1:128:M=32 m32r3_old:0:3:1024:M=32,$L m32r3:0:3:1024:M=32 m64r1_old:0:1:128:M=64,$L m64r1:0:1:128:M=64 m128r1_old:0:1:128:M=128,$L m128r1:0:1:128:M=128 m8r1_old:0:1:128:M=8,$L m8r1:0:1:128:M=8 \
  > $OUT/ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fuzz" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x > $OUT/fuzz.log 2>&1; echo "exit $?" >> $OUT/fuzz.log
