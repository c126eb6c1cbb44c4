mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 600 python tools/abx.py --libs build/variants/lib_head2.so,$L --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x4096,22016x4096,4096x11008 --m 16 --launches 20 --rounds 5 > gpurun_out/r4p_abx_lop3.jsonl 2>&1
timeout 600 python tools/abx.py --libs build/variants/lib_head2.so,$L --shapes 10240x8192,8192x8192,57344x8192,8192x28672 --m 1 --launches 20 --rounds 5 >> gpurun_out/r4p_abx_lop3.jsonl 2>&1
timeout 600 python tools/abx.py --libs build/variants/lib_head2.so,$L --shapes 8192x8192,57344x8192,8192x28672,4096x4096 --m 512,2048 --launches 5 --rounds 5 > gpurun_out/r4p_abx_lop3_prefill.jsonl 2>&1
for v in head2 base; do
  if [ $v == base ]; then unset LPQT_LIB; else export LPQT_LIB=build/variants/lib_$v.so; fi
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 > gpurun_out/r4p_bench70_$v.log 2>&1
  timeout 300 python bench.py --no-cpu-baseline --no-extras --steps 1000 --model llama2-7b > gpurun_out/r4p_bench7_$v.log 2>&1
done
