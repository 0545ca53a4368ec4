#!/bin/bash
# One gpurun call: tests, smoke, bench (+ reference arm), engine A/B, sweeps (perf + the
# reference's csv schema), launch list and ncu --set full captures of the top kernels, ORDERED
# timing, timeline, size scan.
#   gpurun --timeout 3000 -- 'bash tools/gpu_round.sh TAG'
TAG=${1:-r2}
OUT=gpurun_out/$TAG
mkdir -p $OUT
nvidia-smi > $OUT/nvidia-smi.txt 2>&1
nproc > $OUT/nproc.txt; lscpu | grep -i "model name" >> $OUT/nproc.txt
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
if [ "${TESTS:-1}" = "1" ]; then
  timeout 1500 python -m pytest tests -m gpu -q -rA -s > $OUT/pytest_gpu.log 2>&1; echo "pytest exit $?" >> $OUT/pytest_gpu.log
fi
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke exit $?" >> $OUT/smoke.log
timeout 600 python bench.py > $OUT/bench.json 2> $OUT/bench.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 1 > $OUT/bench_reference.json 2> $OUT/bench_reference.err
timeout 600 python tools/ab.py --out $OUT/ab.json async:4:1:1024 tma:1:1:1024 regs:3:1:1024 tc05:2:1:1024 async_ordered:4:1:1024:FIN=ordered probe:0:1:1:PROBE=1 > $OUT/ab.txt 2>&1
timeout 600 python tools/ab.py --n 268435456 --rounds 3 --reps 5 --out $OUT/ab_m.json m2r1:0:1:128:M=2 m2r4:0:4:128:M=2 m4r1:0:1:128:M=4 m4r4:0:4:128:M=4 m4r1b1024:0:1:1024:M=4 m8r1:0:1:128:M=8 m8r4:0:4:128:M=8 m16r1:0:1:128 m16r4:0:4:128 m32r1:0:1:128:M=32 m64r1:0:1:128:M=64 m128r1:0:1:128:M=128 m256r1:0:1:128:M=256 m512r1:0:1:128:M=512 m1024r1:0:1:128:M=1024 m2048r1:0:1:128:M=2048 m4r5b32:0:5:32:M=4 > $OUT/ab_m.txt 2>&1
timeout 1500 python tools/sweep.py --out $OUT/sweep.json > $OUT/sweep.log 2>&1
timeout 900 oracle/_ref/ref_tests_b200 > $OUT/ref_unit_tests.txt 2>&1
timeout 900 oracle/_ref/ref_acceptance_b200 > $OUT/ref_acceptance.txt 2>&1
timeout 600 python tools/ordered_timing.py > $OUT/ordered_timing.txt 2>&1
timeout 300 python tools/ordered_one.py > $OUT/ordered_one.txt 2>&1
if [ "${NCU:-1}" = "1" ]; then
  timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
     python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > $OUT/ncu_launch_bench.log 2>&1
  # reports stay on the box (/tmp): only their raw-page exports travel back (gpurun_out <= 64 MiB)
  cap() {  # name kernel-regex skip count command...
    name=$1; k=$2; sk=$3; cn=$4; shift 4
    timeout 600 ncu -f --set full --clock-control none --import-source on -k regex:$k -s $sk -c $cn -o /tmp/$name "$@" > $OUT/ncu_$name.log 2>&1
    ncu -i /tmp/$name.ncu-rep --page raw --csv > $OUT/$name.raw.csv 2>> $OUT/ncu_$name.log
    ncu -i /tmp/$name.ncu-rep --page source --csv --print-source sass 2>> $OUT/ncu_$name.log | gzip > $OUT/$name.source.csv.gz
  }
  cap async sp_async 3 1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-comparators
  cap tma sp_bulk 3 1 python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu --no-comparators --engine 1
  cap genm_m4_reg gm4_reg 1 1 python tools/ncu_one.py --m 4 --R 1 --B 128 --n 268435456
  cap ordered ordered_ 4 4 python tools/ordered_one.py 16:1:1024:30
fi
timeout 600 python tools/f32_probe.py > $OUT/f32_probe.txt 2>&1
timeout 300 python tools/timeline.py > $OUT/timeline.txt 2>&1
timeout 300 python tools/size_scan.py > $OUT/size_scan.txt 2>&1
echo done > $OUT/DONE
