mkdir -p gpurun_out/s19
timeout 900 python tools/f32_ab.py build_ab/lib_w512.so > gpurun_out/s19/f32_ab.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "fp32 or from_single or m4_register or fuzz" > gpurun_out/s19/pytest.log 2>&1; echo "pytest exit $?" >> gpurun_out/s19/pytest.log
