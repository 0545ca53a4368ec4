OUT=gpurun_out/tr4; mkdir -p $OUT
S=TCR_GM_TR8_SINGLE=1
timeout 300 compute-sanitizer --tool memcheck --error-exitcode 9 python -c "
import torch, paper_2001_05585_b200 as T
x = T.generate('integers', 3, 1 << 20, device=torch.device('cuda', 0))
for m, R, B in ((8,1,128),(8,2,128),(8,4,128),(8,1,1024),(4,1,128),(2,1,128),(32,1,128),(64,2,128)):
    o = T.reduce(x, T.ReductionConfig(m=m, R=R, B=B)); print(m, R, B, o.value)
" > $OUT/memcheck.txt 2>&1; echo "exit $?" >> $OUT/memcheck.txt
timeout 900 python tools/ab.py --n 268435456 --rounds 5 --reps 5 \
  m8r1_old:0:1:128:M=8,$S m8r1:0:1:128:M=8 m8r1k_old:0:1:1024:M=8,$S m8r1k:0:1:1024:M=8 m8r2_old:0:2:128:M=8,$S m8r2:0:2:128:M=8 m8r4_old:0:4:128:M=8,$S m8r4:0:4:128:M=8 m8r3:0:3:128:M=8 \
  > $OUT/ab.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x -k "not fuzz" > $OUT/pytest.log 2>&1; echo "exit $?" >> $OUT/pytest.log
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x > $OUT/fuzz.log 2>&1; echo "exit $?" >> $OUT/fuzz.log
