mkdir -p gpurun_out/s17
timeout 900 python -m pytest tests -m gpu -q -x -k "m4_register" > gpurun_out/s17/pytest_m4.log 2>&1; echo "pytest exit $?" >> gpurun_out/s17/pytest_m4.log
for t in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/s17/san_$t.txt 2>&1; echo "exit $?" >> gpurun_out/s17/san_$t.txt
done
