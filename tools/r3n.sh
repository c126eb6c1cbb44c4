mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $L,build/variants/lib_pro1.so,build/variants/lib_pro2.so --shapes 10240x8192,8192x8192,57344x8192,12288x4096,4096x4096,4096x11008 --m 16 --launches 20 --rounds 5 > gpurun_out/r3n_abx_prologue12.jsonl 2>&1
timeout 900 python bench.py > gpurun_out/r3n_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r3n_launches.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline --no-extras > gpurun_out/r3n_ncu_launch.log 2>&1
