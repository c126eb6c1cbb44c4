mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
python tools/abx.py --libs $L,$L,$L,$L,$L --flags 0,2,2,4,4 --splits 0,0,2,2,4 --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 1,16 --launches 20 --rounds 5 > gpurun_out/r2v_sched.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2v_launches.csv python bench.py --steps 20 --warmup 3 --burn-in 0 --no-cpu-baseline --no-extras > gpurun_out/r2v_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 4 -c 4 -o gpurun_out/r2v_step70b python tools/profile_step.py --model llama2-70b > gpurun_out/r2v_ncu_step.log 2>&1
