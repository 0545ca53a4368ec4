mkdir -p gpurun_out/s10
timeout 900 python tools/ab.py --n 268435456 --rounds 7 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4new:0:1:128:M=4 m4b32old:0:1:32:M=4 m4b32new:0:1:32:M=4,TCR_GM_NAT_ALT=10 m4b64old:0:1:64:M=4 m4b64new:0:1:64:M=4,TCR_GM_NAT_ALT=10 m4b1024:0:1:1024:M=4 m4b256:0:1:256:M=4 m16r1:0:1:128 > gpurun_out/s10/ab28.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s10/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s10/pytest_gpu.log
