mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/r4o_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/r4o_pytest.log
timeout 300 python bench.py > gpurun_out/r4o_bench.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 --model llama2-7b > gpurun_out/r4o_bench7.log 2>&1
