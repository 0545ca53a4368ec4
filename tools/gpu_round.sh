#!/bin/bash
# One gpurun call: tests, smoke, bench, launch list and one ncu --set full capture.
# Usage (from this container): gpurun --timeout 1500 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r1}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nvidia-smi --query-gpu=index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap --format=csv,noheader,nounits > $OUT/clocks_probe.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -i "model name" >> $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 120 python tools/tc05_probe.py > $OUT/tc05_probe.log 2>&1; echo "probe exit $?" >> $OUT/tc05_probe.log
timeout 900 python -m pytest tests -m gpu -q -rA -s > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py --engine 1 > $OUT/bench_mma.json 2> $OUT/bench_mma.err
timeout 600 python bench.py --engine 2 --no-e2e --no-cpu > $OUT/bench_tc05.json 2> $OUT/bench_tc05.err
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch_bench.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sp16_kernel -s 2 -c 1 \
     -o $OUT/sp16 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators --engine 1 > $OUT/ncu_full.log 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc05_kernel -s 2 -c 1 \
     -o $OUT/tc05 python bench.py --steps 2 --warmup 2 --no-e2e --no-cpu --no-comparators --engine 2 > $OUT/ncu_full_tc05.log 2>&1
fi
echo done > $OUT/DONE
