mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "split or fixup or streamk or cluster or workspace or baseline_shapes or llama or fgq or w4a16 or block_params" > gpurun_out/r2f_pytest.log 2>&1; echo "exit $?" >> gpurun_out/r2f_pytest.log
python tools/abx.py --libs build/variants/lib_pf0.so,paper_2312_08583_b200/liblpqt_b200.so --shapes 57344x8192,8192x28672,10240x8192,8192x8192,22016x4096,12288x4096,4096x11008,4096x4096 --m 16,1 > gpurun_out/r2f_abx.log 2>&1
timeout 300 python bench.py --no-extras --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/r2f_bench70.log
timeout 300 python bench.py --model llama2-7b --no-extras --no-cpu-baseline 2>&1 | grep '^{' > gpurun_out/r2f_bench7.log
