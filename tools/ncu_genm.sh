OUT=gpurun_out/ncux; mkdir -p $OUT
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gm_nat -s 2 -c 1 -o $OUT/genm_m4 python bench.py --elems 268435456 --m 4 --R 1 --B 128 --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators > $OUT/l1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gm_tr -s 2 -c 1 -o $OUT/genm_m32 python bench.py --elems 268435456 --m 32 --R 1 --B 128 --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators > $OUT/l2.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:gm_wide_cluster -s 2 -c 1 -o $OUT/genm_m1024_cluster python bench.py --elems 268435456 --m 1024 --R 1 --B 128 --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators > $OUT/l3.log 2>&1
echo done > $OUT/DONE
