mkdir -p gpurun_out/s23
timeout 900 python -m pytest tests -m gpu -q -x -k "m4_register" > gpurun_out/s23/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s23/pytest.log
