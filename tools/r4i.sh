mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/r4i_gpu_tests.log 2>&1; echo "exit $?" >> gpurun_out/r4i_gpu_tests.log
timeout 120 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r4i_smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/r4i_bench.log 2>&1; echo "exit $?" >> gpurun_out/r4i_bench.log
