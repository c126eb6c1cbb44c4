mkdir -p gpurun_out
cat > /tmp/one.py <<'PY'
import sys, torch
sys.path.insert(0, ".")
import paper_2312_08583_b200 as L
n, k, m = (int(v) for v in sys.argv[1:4])
W = (torch.randn(n, k, device="cuda") * 0.02).half()
lin = L.Fp6Linear.from_dense(W)
x = torch.randn(m, k, device="cuda").half()
print("plan", L.plan(m, n, k), flush=True)
y = lin(x); torch.cuda.synchronize()
ref = x.float() @ W.float().t()
print(n, k, m, "ok", float((y.float() - ref).abs().max() / ref.abs().max()), flush=True)
PY
for s in "12288 4096 1" "4096 4096 16" "22016 4096 16" "4096 11008 16" "10240 8192 16" "8192 8192 1" "57344 8192 16" "8192 28672 1"; do
  timeout 30 python /tmp/one.py $s >> gpurun_out/one.log 2>&1 || echo "FAIL/TIMEOUT $s" >> gpurun_out/one.log
done
LPQT_LIB=build/variants/lib_trace.so timeout 60 python tools/trace_run.py --n 12288 --k 4096 --m 1 > gpurun_out/trace_qkv.log 2>&1
