mkdir -p gpurun_out/s9
timeout 900 python tools/ab.py --n 268435456 --rounds 7 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4pf:0:1:128:M=4 m4nopf:0:1:128:M=4,TCR_GM_NAT_ALT=9 m4pf1024:0:1:1024:M=4 m16r1:0:1:128 > gpurun_out/s9/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4pf:0:1:128:M=4 m4nopf:0:1:128:M=4,TCR_GM_NAT_ALT=9 > gpurun_out/s9/ab30.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "m4 or genm or fuzz or from_single or natural or sides" > gpurun_out/s9/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s9/pytest_gpu.log
