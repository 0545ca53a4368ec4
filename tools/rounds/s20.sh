mkdir -p gpurun_out/s20
timeout 300 ncu --metrics gpu__time_duration.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,launch__grid_size,launch__registers_per_thread,launch__occupancy_limit_registers,launch__occupancy_limit_shared_mem --clock-control none --csv --log-file gpurun_out/s20/ord_m4.csv python tools/ordered_one.py 4:1:128:28 > gpurun_out/s20/ord_m4.log 2>&1
timeout 600 ncu -f --set full --clock-control none -k regex:ordered_records -s 1 -c 1 -o /tmp/rec python tools/ordered_one.py 4:1:128:28 > gpurun_out/s20/ncu_rec.log 2>&1
ncu -i /tmp/rec.ncu-rep --page raw --csv > gpurun_out/s20/rec.raw.csv 2>&1
ncu -i /tmp/rec.ncu-rep --page details --csv > gpurun_out/s20/rec.details.csv 2>&1
