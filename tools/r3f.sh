mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs $L,build/variants/lib_ramp10.so,build/variants/lib_ramp20.so,build/variants/lib_ramp35.so --shapes 10240x8192,57344x8192,8192x28672,12288x4096,22016x4096,4096x11008 --m 1,16 --launches 20 --rounds 5 > gpurun_out/r3f_abx_ramp.jsonl 2>&1
for v in ramp10 ramp20 ramp35; do
  LPQT_LIB=build/variants/lib_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 300 --no-extras > gpurun_out/r3f_bench70_$v.log 2>&1
  LPQT_LIB=build/variants/lib_$v.so timeout 300 python bench.py --no-cpu-baseline --steps 300 --no-extras --model llama2-7b > gpurun_out/r3f_bench7_$v.log 2>&1
done
timeout 300 python bench.py --no-cpu-baseline --steps 300 --no-extras > gpurun_out/r3f_bench70_base.log 2>&1
timeout 300 python bench.py --no-cpu-baseline --steps 300 --no-extras --model llama2-7b > gpurun_out/r3f_bench7_base.log 2>&1
timeout 600 python tools/probe.py --shapes 7b,70b --m 128,256 --sched pair > gpurun_out/r3f_probe_pair_small.jsonl 2>&1
timeout 600 python tools/probe.py --shapes 7b,70b --m 128,256 > gpurun_out/r3f_probe_auto_small.jsonl 2>&1
