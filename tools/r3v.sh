mkdir -p gpurun_out
L=paper_2312_08583_b200/liblpqt_b200.so
timeout 900 python tools/abx.py --libs $L,build/variants/lib_head.so --shapes 10240x8192,8192x8192,57344x8192,8192x28672,12288x4096,4096x11008 --m 512,2048 --launches 10 --rounds 5 > gpurun_out/r3v_abx_fgqpair.jsonl 2>&1
timeout 900 python tools/probe.py --shapes 7b,13b --m 32,64,96,128 --sched single --split 0,2,4,8 > gpurun_out/r3v_probe_split_single.jsonl 2>&1
