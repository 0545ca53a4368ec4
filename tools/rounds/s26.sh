mkdir -p gpurun_out/s26
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/s26/build.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s26/smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/s26/smoke.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/s26/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/s26/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/s26/bench.json 2> gpurun_out/s26/bench.err
