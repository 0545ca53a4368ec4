mkdir -p gpurun_out/s22
timeout 1200 python tools/ab.py --n 268435456 --rounds 7 --reps 10 b32old:0:1:32:M=4,LIB=build_ab/lib_w512.so b32rt:0:1:32:M=4 b128:0:1:128:M=4 b128rt:0:1:128:M=4,TCR_GM_NAT_ALT=11 > gpurun_out/s22/ab28.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "m4_register or fp32 or from_single or fuzz or ordered" > gpurun_out/s22/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s22/pytest.log
