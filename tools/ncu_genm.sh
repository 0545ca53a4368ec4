# ncu --set full captures of the m != 16 engines (one kernel each), n = 2^28, R = 1, B = 128:
#   gpurun --timeout 1200 -- 'bash tools/ncu_genm.sh'   then tools/summarize_profiles.py
OUT=gpurun_out/ncux; mkdir -p $OUT
cap() {  # name kernel-regex m
  timeout 300 ncu --set full --clock-control none --import-source on -k regex:$2 -s 2 -c 1 -o $OUT/genm_$1 \
    python bench.py --elems 268435456 --m $3 --R 1 --B 128 --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators > $OUT/$1.log 2>&1
}
cap m2 gm_nat_fast 2
cap m4 gm_nat_fast 4
cap m8 gm_tr 8
cap m32 gm_tr 32
cap m1024_cluster gm_wide_cluster 1024
echo done > $OUT/DONE
