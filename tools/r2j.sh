mkdir -p gpurun_out
for m in 512 2048; do
timeout 600 ncu --set full --clock-control none --import-source on -k regex:w6a16 -s 2 -c 1 -o gpurun_out/r2j_prefill_m$m python tools/profile_one.py --n 8192 --k 8192 --m $m --iters 3 > gpurun_out/r2j_ncu_m$m.log 2>&1
done
python tools/probe.py --shapes 70b --m 512,2048 > gpurun_out/r2j_probe.log 2>&1
