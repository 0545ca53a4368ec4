mkdir -p gpurun_out/s7
timeout 900 python tools/ab.py --n 268435456 --rounds 7 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4pf:0:1:128:M=4 m4nopf:0:1:128:M=4,TCR_GM_NAT_ALT=9 m4pf1024:0:1:1024:M=4 m4pf256:0:1:256:M=4 m16r1:0:1:128 > gpurun_out/s7/ab28.txt 2>&1
timeout 900 python tools/ab.py --n 1073741824 --rounds 5 --reps 10 m4old:0:1:128:M=4,TCR_GM_NAT_ALT=8 m4pf:0:1:128:M=4 m4nopf:0:1:128:M=4,TCR_GM_NAT_ALT=9 > gpurun_out/s7/ab30.txt 2>&1
