mkdir -p gpurun_out
O=gpurun_out/r5s2_sweeps_nm.jsonl; : > $O
for kind in cgq fgq128 fgq16 fp5 int4_128; do
  timeout 900 python tools/sweep_check.py --sets 7b,70b_tp8,ragged --kind $kind --layout nm --ms 1,16,17,33,64,65,128,256,512,1024 | tail -1 >> $O 2>&1
done
