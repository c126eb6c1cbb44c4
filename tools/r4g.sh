mkdir -p gpurun_out
timeout 1200 python tools/probe.py --shapes sc15b --m 1,4,16,32,64,128,256,512 > gpurun_out/r4g_probe_sc15b.jsonl 2>&1
timeout 1200 python tools/probe.py --shapes 70b_tp2,70b_tp4,70b_tp8 --m 1,16,512 > gpurun_out/r4g_probe_tp_shards.jsonl 2>&1
