mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_streamk_fixup.py -x -q > gpurun_out/r5o_fixup.log 2>&1; echo "rc=$?" >> gpurun_out/r5o_fixup.log
timeout 600 python tools/repro_fgq.py 128 > gpurun_out/r5o_fgq128.jsonl 2>&1
timeout 600 python tools/repro_fgq.py 32 > gpurun_out/r5o_fgq32.jsonl 2>&1
for kind in fgq128 fgq32 fgq16; do
  timeout 600 python tools/sweep_check.py --sets ragged --kind $kind > gpurun_out/r5o_sweep_ragged_$kind.jsonl 2>&1; echo "rc=$?" >> gpurun_out/r5o_sweep_ragged_$kind.jsonl
done
