mkdir -p gpurun_out/s6
timeout 900 python tools/ab.py --n 268435456 --rounds 7 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4new:0:1:128:M=4 m4old32:0:1:32:M=4,TCR_GM_NAT_ALT=8 m4new32:0:1:32:M=4 m4old1024:0:1:1024:M=4,TCR_GM_NAT_ALT=8 m4new1024:0:1:1024:M=4 m16r1:0:1:128 shuffle:0:1:1:SHUFFLE=1 > gpurun_out/s6/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4new:0:1:128:M=4 > gpurun_out/s6/ab30.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s6/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s6/pytest_gpu.log
