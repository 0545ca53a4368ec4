mkdir -p gpurun_out/s27
timeout 900 python tools/ab.py --rounds 5 --reps 5 old:0:1:1024:FIN=ordered,LIB=build_ab/lib_pre_seed.so new:0:1:1024:FIN=ordered > gpurun_out/s27/u30.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "ordered or seeded or permutation or oracle64 or golden" > gpurun_out/s27/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s27/pytest.log
timeout 600 python tools/ordered_timing.py > gpurun_out/s27/ordered_timing.txt 2>&1
