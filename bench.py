"""bench.py — W6A16 (FP6 e3m2 weight, FP16 activation) linear on B200.

Workload (N=1, the north-star target, BASELINE.json configs[3] at TP=1): one
LLaMA-2-70B decoder block's four linear layers (QKV 10240x8192, O 8192x8192,
gate_up 57344x8192, down 8192x28672) at decode batch M (default 16).  A
"step" = those four W6A16 GEMMs over one batch.  Synthetic data: random-init
N(0, 0.02) weights quantized on the GPU, N(0, 1) fp16 activations.  Extra
device-timed lines ride along: the same step at M = 1 and the LLaMA-2-7B step
(configs[1]) at M = 16 (`--no-extras` skips them; `--model llama2-7b` makes
7B the headline).

Metric (BASELINE.json): "W6A16 linear TFLOPS & weight HBM GB/s vs roofline
and cuBLAS FP16, batch 1-512" -> value = algorithmic HBM GB/s of the step
(FP6 planes 0.75 B/weight + 2 B/row scales + fp16 X + fp16 Y); TFLOPS,
cuBLAS fp16 and the roofline fraction ride along.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--m 16] [--model llama2-70b|llama2-7b]
                  [--impl ours|reference]

N>1 (torchrun): column-sharded tensor parallelism: every rank
holds N/P rows of every layer, runs its shard GEMM, and one NCCL
all_gather_into_tensor per layer assembles Y[N, M] -> "scaling": "strong".

Timing: W untimed warm-up steps, then EXACTLY K steps replayed from CUDA
graphs, bracketed by barrier + synchronize, device-timed with CUDA events,
max over ranks.  L2: the step's weights (646 MB FP6 at 70B, 151 MB at 7B) are
rotated over >= 2 distinct copies (> 2 x 126 MB L2), so every step reads cold
weights.  cpu_baseline / --impl reference: the reference package itself
(baseline/_ref, tools/install_reference.sh) on a bounded row sample.
"""

from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LAYERS_7B = [("qkv", 12288, 4096), ("o", 4096, 4096), ("gate_up", 22016, 4096), ("down", 4096, 11008)]
LAYERS_70B = [("qkv", 10240, 8192), ("o", 8192, 8192), ("gate_up", 57344, 8192), ("down", 8192, 28672)]
METRIC = "W6A16 linear TFLOPS & weight HBM GB/s vs roofline and cuBLAS FP16, batch 1-512"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return {"hbm_gbs": float(d["hbm_gbs"]), "bf16_tflops": float(d["bf16_tflops"]),
                "bf16_tflops_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return dict(FALLBACK_PEAKS, bf16_tflops_sustained=FALLBACK_PEAKS["bf16_tflops"],
                source="fallback (B200_PROFILING.md)")


def step_bytes(layers, m):
    """Algorithmic bytes of one step: FP6 planes + f16 row scales + X + Y (fp16)."""
    tot = 0
    for _, n, k in layers:
        nk = n * k
        seg4 = ((nk + 1) // 2 + 3) // 4 * 4
        seg2 = ((2 * nk + 7) // 8 + 3) // 4 * 4
        tot += seg4 + seg2 + 2 * n + 2 * m * k + 2 * m * n
    return tot


def sample_bytes(layers, m, rows):
    """The share of the step's algorithmic bytes a row sample covers: each
    layer's bytes x rows / N (X and the scales amortised with the rows)."""
    return sum(layer_bytes(n, k, m) * min(rows, n) / n for _, n, k in layers)


def layer_bytes(n, k, m):
    return step_bytes([("", n, k)], m)


def step_flops(layers, m):
    return sum(2 * m * n * k for _, n, k in layers)


# ---------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 100 ms while active."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 8:
                self.rows.append(parts)

    def __exit__(self, *exc):
        if self.proc is not None:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[4 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------
def setup_dist(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    elif torch.cuda.is_available():
        torch.cuda.set_device(0)
    return world, rank, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(x, world):
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def build_layers(layers, world, rank, copies, seed=0):
    """Quantize + prepack each layer's row shard on the GPU; `copies` distinct
    weight sets for L2 rotation.  Returns list[copy] of list[Fp6Weight]."""
    import torch
    import paper_2312_08583_b200 as L
    from paper_2312_08583_b200.tp import shard_rows
    g = torch.Generator(device="cuda").manual_seed(seed + 1000 * rank)
    sets = []
    for _ in range(copies):
        ws = []
        for _, n, k in layers:
            a, b = shard_rows(n, world, rank)
            W = (torch.randn(b - a, k, generator=g, device="cuda") * 0.02).half()
            ws.append(L.Fp6Weight.quantize(W, bias_shift=True))
            del W
        sets.append(ws)
    torch.cuda.synchronize()
    return sets


def run_ours(args, world, rank, layers, m, e2e=True, burn_in=None):
    import torch
    import paper_2312_08583_b200 as L
    from paper_2312_08583_b200 import _lib

    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    fp6_set = step_bytes(layers, 0) // world
    copies = max(2, -(-2 * l2 // max(fp6_set, 1)))
    sets = build_layers(layers, world, rank, copies)

    gen = torch.Generator(device="cuda").manual_seed(7)
    xs = [torch.randn(k, m, generator=gen, device="cuda").half() for _, _, k in layers]   # X[K, M]
    xts = [x.t().contiguous() for x in xs]                                                # K-major operand
    shard_n = [sets[0][i].n for i in range(len(layers))]
    ys = [torch.empty(n_local, m, device="cuda", dtype=torch.float16) for n_local in shard_n]
    yfull = [torch.empty(n, m, device="cuda", dtype=torch.float16) for _, n, _ in layers]
    lib = _lib.load()

    def next_of(c, i):
        # the linear that runs next on the stream: the step's next layer, or
        # the first layer of the next step (the next weight copy)
        if args.no_l2_next:
            return None
        return sets[c][i + 1] if i + 1 < len(layers) else sets[(c + 1) % copies][0]

    def launch(i, w, nxt=None):
        # reference layout Y[N_p, M] (gemm.py:65), fp16 out
        ws_bytes = int(lib.lpqt_w6a16_workspace_bytes(m, w.n, w.k, 0))
        ws = _lib.Workspace.get(ws_bytes) if ws_bytes else None
        # programmatic dependent launch: the weights are static, so each GEMM
        # streams its weight tiles while the previous layer's kernel drains;
        # and its drain pulls the next linear's first weight bytes into L2
        pf = None if nxt is None else _lib.NextLinear(nxt.tiles.data_ptr(), m, nxt.n, nxt.k, 0, 0, args.pf_bytes)
        _lib.check(lib.lpqt_w6a16_linear_pf(w.tiles.data_ptr(), w.scales.data_ptr(), xts[i].data_ptr(), w.k, m,
                                            w.n, w.k, ys[i].data_ptr(), _lib.F16, _lib.Y_NM, m, 0, _lib.ptr(ws),
                                            ws.numel() if ws is not None else 0, _lib.LAUNCH_PDL,
                                            None if pf is None else ctypes.byref(pf), _lib.stream_ptr()))

    def step(c):
        for i, w in enumerate(sets[c]):
            launch(i, w, next_of(c, i))
            if world > 1:
                import torch.distributed as dist
                dist.all_gather_into_tensor(yfull[i], ys[i])

    # warm-up (also allocates the workspace before capture)
    for s in range(max(args.warmup, 1)):
        step(s % copies)
    torch.cuda.synchronize()

    # one graph per weight copy (the timed region: back-to-back launches, PDL
    # edges between consecutive GEMMs), plus one per copy with external
    # events between the launches for the per-launch breakdown (serialised)
    def capture(c, with_events):
        evs = [torch.cuda.Event(enable_timing=True, external=True) for _ in range(len(layers) + 1)]
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for i, w in enumerate(sets[c]):
                if with_events:
                    evs[i].record()
                launch(i, w, None if with_events else next_of(c, i))
                if world > 1:
                    import torch.distributed as dist
                    dist.all_gather_into_tensor(yfull[i], ys[i])
            if with_events:
                evs[-1].record()
        return g, evs

    graphs = [capture(c, False)[0] for c in range(copies)]
    # the timed region replays graphs of G consecutive steps (step j uses weight
    # copy j % copies): PDL edges then also join the last GEMM of a step to
    # the first of the next inside a graph, as a graph-captured serving loop
    # does; K = q G + r steps = q replays of the G-step graph + r one-step graphs
    G = max(copies, args.graph_steps // copies * copies) if args.graph_steps > 1 else 1
    multi = None
    if G > 1:
        multi = torch.cuda.CUDAGraph()
        with torch.cuda.graph(multi):
            for j in range(G):
                for i, w in enumerate(sets[j % copies]):
                    launch(i, w, next_of(j % copies, i))
                    if world > 1:
                        import torch.distributed as dist
                        dist.all_gather_into_tensor(yfull[i], ys[i])

    def run_steps(k):
        q, r = (k // G, k % G) if multi is not None else (0, k)
        for _ in range(q):
            multi.replay()
        for s in range(r):
            graphs[s % copies].replay()

    run_steps(args.warmup)
    torch.cuda.synchronize()

    # burn-in so the clock sampler sees the part under load, then the timed region
    launches_before = _lib.launch_count()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", "0"))) as clk:
        t_end = time.time() + (args.burn_in if burn_in is None else burn_in)
        while time.time() < t_end:
            run_steps(max(G, copies))
            torch.cuda.synchronize()
        barrier(world)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        run_steps(args.steps)
        e1.record()
        torch.cuda.synchronize()
        barrier(world)
    t_local = e0.elapsed_time(e1) * 1e-3
    t = max_over_ranks(t_local, world)
    gpu_launches = args.steps * len(layers)          # kernel nodes per replayed graph x replays
    assert _lib.launch_count() == launches_before     # replays, no new host launches

    # per-launch durations (serialised by the events; informational)
    timed = [capture(c, True) for c in range(copies)]
    for r in range(4):
        for g, _ in timed:
            g.replay()
    torch.cuda.synchronize()
    per_layer = []
    for i, (name, n, k) in enumerate(layers):
        d = statistics.mean(ev[i].elapsed_time(ev[i + 1]) * 1e-3 for _, ev in timed)
        nb = layer_bytes(sets[0][i].n, k, m)
        per_layer.append({"layer": name, "n": sets[0][i].n, "k": k, "us": round(d * 1e6, 2),
                          "GBps": round(nb / d / 1e9, 1), "plan": L.plan(m, sets[0][i].n, k)})
    del timed

    total_bytes = step_bytes(layers, m)       # whole job (all ranks)
    value = total_bytes * args.steps / t / 1e9
    res = {"t": t, "value": value, "per_layer": per_layer, "gpu_launches": gpu_launches,
           "clocks": clk.summary(), "copies": copies, "graph_steps": G}

    # cuBLAS fp16 comparator on the same step (fp16 weights, same shards)
    if rank == 0 or world > 1:
        res["cublas"] = time_cublas(layers, world, rank, m, args)
    # e2e through the public API with host buffers
    if e2e:
        res["e2e"] = time_e2e(layers, sets[0], world, rank, m, args)
    del sets, graphs
    torch.cuda.empty_cache()
    return res


def time_quantize(layers, args):
    """K1 on the GPU: RTN FP6 CGQ quantize of the step's four fp16 weights,
    (a) the reference API `quantize_tensor(W, CGQ FP6, bias_shift=True)` ->
    canonical 4+2 planes + scales + folded scales (quantizer.py:189-248) and
    (b) `Fp6Weight.quantize` straight into the GEMM's tile layout.  Device
    time (CUDA events), median of 5; algorithmic bytes = the fp16 weights
    read twice (row peaks, encode) + 0.75 B per weight written."""
    import torch
    import paper_2312_08583_b200 as L
    cgq = L.QuantScheme(L.Granularity.CGQ, L.TensorFormat.FP6_E3M2)
    g = torch.Generator(device="cuda").manual_seed(11)
    ws = [(torch.randn(n, k, generator=g, device="cuda") * 0.02).half() for _, n, k in layers]
    nw = sum(w.numel() for w in ws)

    def timed(fn):
        fn()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e-3)
        return sorted(ts)[2]
    t_api = timed(lambda: [L.quantize_tensor(w, cgq, bias_shift=True) for w in ws])
    t_tiles = timed(lambda: [L.Fp6Weight.quantize(w) for w in ws])
    byts = nw * (2 * 2 + 0.75)
    del ws
    torch.cuda.empty_cache()
    return {"workload": f"{args.model} quantize (RTN FP6 CGQ + 4+2 pack + fold) of the step's four weights, fp16 in",
            "value": round(byts / t_api / 1e9, 1), "unit": "GB/s", "weights": nw,
            "ms": round(t_api * 1e3, 3), "Mweights_per_s": round(nw / t_api / 1e6, 1),
            "api": "paper_2312_08583_b200.quantize_tensor(W_cuda, CGQ FP6, bias_shift=True) -> canonical planes",
            "tiles_path": {"ms": round(t_tiles * 1e3, 3), "GBps": round(byts / t_tiles / 1e9, 1),
                           "api": "Fp6Weight.quantize (straight into the GEMM tile layout)"},
            "note": "device time; compare cpu_baseline.quantize_weights_per_s (the reference's numpy quantize)"}


def time_cublas(layers, world, rank, m, args):
    import torch
    from paper_2312_08583_b200.tp import shard_rows
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    f16_set = sum(2 * n * k for _, n, k in layers) // world
    copies = max(1, -(-2 * l2 // f16_set))
    g = torch.Generator(device="cuda").manual_seed(11)
    wsets = []
    for _ in range(copies):
        wsets.append([(torch.randn(*(lambda ab: (ab[1] - ab[0], k))(shard_rows(n, world, rank)), generator=g,
                                   device="cuda") * 0.02).half() for _, n, k in layers])
    xs = [torch.randn(m, k, generator=g, device="cuda").half() for _, _, k in layers]
    outs = [None] * len(layers)

    def step(c):
        for i, W in enumerate(wsets[c]):
            outs[i] = torch.matmul(xs[i], W.t())

    for c in range(copies):
        step(c)
    torch.cuda.synchronize()
    graphs = []
    for c in range(copies):
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            step(c)
        graphs.append(gr)
    for s in range(max(args.warmup, 3)):
        graphs[s % copies].replay()
    torch.cuda.synchronize()
    steps = max(args.steps // 2, 50)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for s in range(steps):
        graphs[s % copies].replay()
    e1.record()
    torch.cuda.synchronize()
    t = e0.elapsed_time(e1) * 1e-3 / steps
    f16_bytes = sum(2 * n * k + 2 * m * k + 2 * m * n for _, n, k in layers) // world
    del wsets
    torch.cuda.empty_cache()
    return {"ms_per_step": round(t * 1e3, 4), "GBps_fp16_weights": round(f16_bytes / t / 1e9, 1),
            "TFLOPS": round(step_flops(layers, m) / world / t / 1e12, 2), "copies": copies}


def time_e2e(layers, wset, world, rank, m, args):
    """Same metric end to end through the public serving API with host
    buffers: every step copies the step's activations (all four layers' x
    [M, K] fp16, from one pinned buffer) host -> device, runs `w6a16_linear`
    per layer (torch layout, fp16 out; under TP followed by the all-gather),
    and reads all outputs y [M, N] fp16 back into one pinned host buffer; the
    host waits for the results every step.  Copies run per layer on two copy
    streams so they overlap the linears.  The step's calls are captured once
    in a CUDA graph (as a serving loop would) and replayed."""
    import torch
    from paper_2312_08583_b200.linear import w6a16_linear
    ks = [k for _, _, k in layers]
    ns = [n for _, n, _ in layers]
    xoff = np.cumsum([0] + [m * k for k in ks])
    yoff = np.cumsum([0] + [m * n for n in ns])
    xh = torch.randn(int(xoff[-1])).half().pin_memory()
    yh = torch.empty(int(yoff[-1]), dtype=torch.float16).pin_memory()
    xd = torch.empty_like(xh, device="cuda")
    yd = torch.empty(int(yoff[-1]), dtype=torch.float16, device="cuda")
    ys_local = [torch.empty(m, w.n, dtype=torch.float16, device="cuda") for w in wset]

    # copies overlap the compute: layer i's x arrives on a copy stream while
    # earlier layers run, and y[i] leaves on another as soon as layer i is
    # done; the step ends when the last y is on the host
    s_h2d, s_d2h = torch.cuda.Stream(), torch.cuda.Stream()
    n_l = len(wset)
    ev_x = [torch.cuda.Event() for _ in range(n_l)]
    ev_y = [torch.cuda.Event() for _ in range(n_l)]
    ev_start, ev_d2h = torch.cuda.Event(), torch.cuda.Event()

    def body():
        cur = torch.cuda.current_stream()
        ev_start.record(cur)
        s_h2d.wait_event(ev_start)
        with torch.cuda.stream(s_h2d):
            for i in range(n_l):
                xd[int(xoff[i]):int(xoff[i + 1])].copy_(xh[int(xoff[i]):int(xoff[i + 1])], non_blocking=True)
                ev_x[i].record(s_h2d)
        for i, w in enumerate(wset):
            x = xd[int(xoff[i]):int(xoff[i + 1])].view(m, ks[i])
            y = yd[int(yoff[i]):int(yoff[i + 1])].view(m, ns[i])
            nxt = wset[(i + 1) % len(wset)]    # the next linear on the stream (L2 prefetch hint)
            cur.wait_event(ev_x[i])
            if world == 1:
                w6a16_linear(x, w, out=y, prefetch=nxt)
            else:
                import torch.distributed as dist
                w6a16_linear(x, w, out=ys_local[i], prefetch=nxt)
                # column shards gathered along N: [P, M, N/P] -> y[M, N]
                parts = torch.empty(world, m, w.n, dtype=torch.float16, device="cuda")
                dist.all_gather_into_tensor(parts, ys_local[i])
                y.copy_(parts.permute(1, 0, 2).reshape(m, ns[i]))
            ev_y[i].record(cur)
            s_d2h.wait_event(ev_y[i])
            with torch.cuda.stream(s_d2h):
                yh[int(yoff[i]):int(yoff[i + 1])].copy_(yd[int(yoff[i]):int(yoff[i + 1])], non_blocking=True)
        ev_d2h.record(s_d2h)
        cur.wait_event(ev_d2h)

    for _ in range(3):
        body()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        body()
    for _ in range(max(args.warmup, 3)):
        g.replay()
        torch.cuda.synchronize()
    steps = max(min(args.steps, 500), 20)
    barrier(world)
    t0 = time.perf_counter()
    for _ in range(steps):
        g.replay()
        torch.cuda.synchronize()   # the host has the step's results
    t = time.perf_counter() - t0
    t = max_over_ranks(t, world)
    return {"value": round(step_bytes(layers, m) * steps / t / 1e9, 2), "unit": "GB/s",
            "h2d_bytes_per_step": int(xh.numel() * 2), "d2h_bytes_per_step": int(yh.numel() * 2),
            "ms_per_step": round(t / steps * 1e3, 4),
            "api": "paper_2312_08583_b200.w6a16_linear per layer (torch layout, fp16 in/out): pinned host x -> "
                   "device, four linears, y -> pinned host each step, host sync per step; per-layer copies on "
                   "two copy streams overlap the linears; the step's calls captured once in a CUDA graph and "
                   "replayed"}


# ---------------------------------------------------------------------------
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The UNMODIFIED reference package (lpqt 0.1.0) installed in baseline/_ref
    by tools/install_reference.sh (pip --target; git-ignored, travels to the
    GPU box).  None when it is not staged (then the oracle port stands in)."""
    if not os.path.isdir(os.path.join(REF_DIR, "lpqt")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import lpqt
    assert os.path.dirname(os.path.dirname(os.path.abspath(lpqt.__file__))) == REF_DIR, lpqt.__file__
    return lpqt


class _PortAsRef:
    """The oracle restatement behind the reference's call signatures (used only
    when baseline/_ref is absent)."""

    def __init__(self):
        from oracle import lpqt_oracle as O
        self.O = O

    def quantize(self, W):
        return self.O.quantize_tensor(W, bias_shift=True)

    def gemm(self, q, X):
        n = q["scales"].size
        return self.O.gemm_quantized(q["codes"], q["scales"], n, q["codes"].size // max(n, 1), X)


class _Ref:
    def __init__(self, lpqt):
        self.lpqt = lpqt
        self.scheme = lpqt.QuantScheme(lpqt.Granularity.CGQ, lpqt.TensorFormat.FP6_E3M2)

    def quantize(self, W):
        # quantize_tensor(W.astype(float64), CGQ FP6, bias_shift=True)
        return self.lpqt.quantize_tensor(W.astype(np.float64), self.scheme, bias_shift=True)

    def gemm(self, q, X):
        return self.lpqt.gemm_quantized(q, X)


def reference_impl():
    lp = load_reference()
    return (_Ref(lp), "reference") if lp is not None else (_PortAsRef(), "port")


def _sample_inputs(layers, m, rows, seed):
    """BASELINE.md §3 inputs on a row sample: W = N(0,1)*0.02 f32 -> fp16 (the
    first `rows` rows of each layer), X = N(0,1) [K, M] fp16."""
    out = []
    for i, (_, n, k) in enumerate(layers):
        rng = np.random.default_rng(seed + i)
        W = (rng.standard_normal((rows, k), dtype=np.float32) * 0.02).astype(np.float16)
        X = np.random.default_rng(seed + 100 + i).standard_normal((k, m)).astype(np.float16)
        out.append((W, X))
    return out


def cpu_baseline(layers, m, budget_s=15.0):
    """The reference's own CPU path (baseline/_ref lpqt: quantize_tensor +
    gemm_quantized, quantizer.py:189-248 / gemm.py:65-94) timed on this
    host, single process (numpy elementwise, effectively one core), on a
    bounded sample: the first R rows of each of the step's layers.
    `value` = algorithmic GB/s of gemm_quantized over the sample (the
    metric's unit); the quantize rate rides along."""
    impl, kind = reference_impl()
    rows = 64
    sample = _sample_inputs(layers, m, rows, seed=0)
    t0 = time.perf_counter()
    qs = [impl.quantize(W) for W, _ in sample]
    t_quant = time.perf_counter() - t0
    nbytes = sample_bytes(layers, m, rows)
    reps = 0
    t0 = time.perf_counter()
    while True:
        for q, (_, X) in zip(qs, sample):
            impl.gemm(q, X)
        reps += 1
        if time.perf_counter() - t0 > budget_s:
            break
    t = time.perf_counter() - t0
    n_weights = sum(rows * k for _, _, k in layers)
    return {"value": round(nbytes * reps / t / 1e9, 5), "unit": "GB/s", "cores": 1, "kind": kind,
            "quantize_weights_per_s": round(n_weights / t_quant, 1),
            "sample": f"{'reference lpqt 0.1.0 (baseline/_ref)' if kind == 'reference' else 'oracle port'}: "
                      f"quantize_tensor (CGQ FP6, bias_shift) of the first {rows} rows of each of the "
                      f"{len(layers)} layers ({n_weights} weights, {t_quant:.2f}s), then gemm_quantized at M={m} "
                      f"on those rows, {reps} reps in {t:.1f}s; single process, numpy"}


def run_reference(args, world, rank):
    """--impl reference: the reference's own CPU implementation (baseline/_ref
    lpqt gemm_quantized) on all host threads, row-parallel over a process pool
    (SPEC.md:373-375 permits row parallelism); each step = every worker's
    gemm_quantized over its row sample of each layer."""
    import multiprocessing as mp
    layers = LAYERS_7B if args.model == "llama2-7b" else LAYERS_70B
    m = args.m
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    rows_per_worker = 16
    with mp.get_context("fork").Pool(cores, initializer=_ref_init, initargs=(layers, m, rows_per_worker)) as pool:
        kinds = set(pool.map(_ref_kind, range(cores)))
        for _ in range(max(args.warmup, 1)):
            pool.map(_ref_step, range(cores))
        t_budget = 120.0
        steps = 0
        t0 = time.perf_counter()
        while steps < args.steps:
            pool.map(_ref_step, range(cores))
            steps += 1
            if time.perf_counter() - t0 > t_budget:
                break
        t = time.perf_counter() - t0
    kind = kinds.pop() if len(kinds) == 1 else "port"
    nbytes = sample_bytes(layers, m, rows_per_worker * cores)
    value = nbytes * steps / t / 1e9
    sample = (f"{'reference lpqt 0.1.0 (baseline/_ref)' if kind == 'reference' else 'oracle port'} "
              f"gemm_quantized on {rows_per_worker} rows x {cores} processes of each {args.model} layer per step, "
              f"M={m}; {steps} steps timed")
    return {"value": value, "t": t, "steps": steps, "cores": cores, "sample": sample, "kind": kind}


_REF = {}


def _ref_init(layers, m, rows):
    impl, kind = reference_impl()
    _REF["impl"], _REF["kind"] = impl, kind
    sample = _sample_inputs(layers, m, rows, seed=os.getpid())
    _REF["work"] = [(impl.quantize(W), X) for W, X in sample]


def _ref_kind(_):
    return _REF["kind"]


def _ref_step(_):
    impl = _REF["impl"]
    for q, X in _REF["work"]:
        impl.gemm(q, X)
    return 0


# ---------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=1000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--m", type=int, default=16, help="decode batch (tokens)")
    ap.add_argument("--model", default="llama2-70b", choices=["llama2-7b", "llama2-70b"])
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--burn-in", type=float, default=1.5, help="seconds of untimed load before timing")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true", help="skip the extra M=1 / 7B lines")
    ap.add_argument("--graph-steps", type=int, default=8, help="steps per replayed CUDA graph")
    ap.add_argument("--no-l2-next", action="store_true", help="no next-linear L2 prefetch hint")
    ap.add_argument("--pf-bytes", type=int, default=0, help="next-linear L2 prefetch bytes per CTA (0: 64 KiB)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    layers = LAYERS_7B if args.model == "llama2-7b" else LAYERS_70B
    workload = f"{args.model} decoder-block linears (QKV/O/gate_up/down) decode M={args.m}"
    config = {"workload": workload, "layers": [f"{n}x{k}" for _, n, k in layers], "batch_m": args.m,
              "baseline_config": "BASELINE.json configs[3] (LLaMA-2-70B shapes; TP degree = n_gpus)"
              if args.model == "llama2-70b" else "BASELINE.json configs[1] (LLaMA-2-7B shapes)",
              "tensor_parallel": world, "parallelism": f"tp{world} column-sharded + NCCL all-gather"
              if world > 1 else "single GPU", "activations": "fp16", "weights": "FP6 e3m2 (4+2), per-row f16 scale",
              "l2_hygiene": "inputs larger than L2: weights rotated over >=2 distinct copies (>2x L2) per step",
              "graph_steps": args.graph_steps}

    if args.impl == "reference":
        if rank != 0:
            return
        r = run_reference(args, world, rank)
        line = {"metric": METRIC, "value": round(r["value"], 6), "unit": "GB/s", "n_gpus": args.gpus,
                "steps": r["steps"], "warmup": args.warmup, "ms_per_step": round(r["t"] / r["steps"] * 1e3, 3),
                "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": config, "impl": "reference",
                "cpu_baseline": {"value": round(r["value"], 6), "unit": "GB/s", "cores": r["cores"],
                                 "kind": r["kind"], "sample": r["sample"]},
                "e2e": {"value": round(r["value"], 6), "unit": "GB/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    world, rank, _ = setup_dist(args)
    peaks = load_peaks()
    m = args.m
    res = run_ours(args, world, rank, layers, m)
    t_step = res["t"] / args.steps
    flops = step_flops(layers, m)
    # roofline of the dominant kernel: the W6A16 GEMM is every launch of the
    # step, so achieved = the step's algorithmic bytes / the timed step time
    # (CUDA events over the timed region, launches back to back)
    achieved = step_bytes(layers, m) / world / t_step / 1e9
    traffic = None
    traffic_note = None
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        with open(tp) as f:
            tr = json.load(f).get(f"{args.model}_m{m}")
        if tr:
            # DRAM bytes (read + write) of the step's launches from one
            # ncu --set full capture, per step like `achieved`
            traffic = tr["bytes_per_step"] // world
            traffic_note = {"traffic_over_algorithmic": tr["ratio"], "source": "profiles/ncu_traffic.json: " +
                            tr["source"]}
    extras = []
    if not args.no_extras:
        # the other north-star decode point (M = 1) and the 7B step (BASELINE
        # configs[1]); device-timed like the headline, no e2e
        for model, mx in ((args.model, 1 if m != 1 else 16), ("llama2-7b" if args.model != "llama2-7b"
                                                                else "llama2-70b", 16), (args.model, 512)):
            lx = LAYERS_7B if model == "llama2-7b" else LAYERS_70B
            import argparse as _ap
            ax_args = _ap.Namespace(**dict(vars(args), steps=args.steps if mx <= 16 else max(20, args.steps // 20)))
            rx = run_ours(ax_args, world, rank, lx, mx, e2e=False, burn_in=0.5)
            tx = rx["t"] / ax_args.steps
            ax = step_bytes(lx, mx) / world / tx / 1e9
            ent = {"workload": f"{model} decoder-block linears {'decode' if mx <= 16 else 'prefill'} M={mx}",
                   "value": round(step_bytes(lx, mx) * ax_args.steps / rx["t"] / 1e9, 2), "unit": "GB/s",
                   "steps": ax_args.steps, "ms_per_step": round(tx * 1e3, 5),
                   "roofline_frac": round(ax / peaks["hbm_gbs"], 4),
                   "tflops": round(step_flops(lx, mx) / world / tx / 1e12, 2),
                   "speedup_vs_cublas_fp16": round(rx["cublas"]["ms_per_step"] / (tx * 1e3), 3),
                   "cublas_fp16_tflops": rx["cublas"]["TFLOPS"],
                   "clocks": rx["clocks"], "per_launch_serialised": rx["per_layer"]}
            if mx > 16:   # prefill: tensor-pipe bound, roofline against the measured dense bf16 peak
                ent["roofline"] = {"bound": "tensor", "achieved": ent["tflops"],
                                   "peak": peaks["bf16_tflops_sustained"], "unit": "TFLOP/s",
                                   "frac": round(ent["tflops"] / peaks["bf16_tflops_sustained"], 4),
                                   "peak_source": peaks["source"] + " (sustained)"}
            extras.append(ent)
        if world == 1:
            extras.append(time_quantize(layers, args))
    if rank != 0:
        return
    line = {
        "metric": METRIC, "value": round(res["value"], 2), "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 5),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "fp16", "dtype_detail": "fp6 e3m2 weights rebuilt to fp16, fp16 activations, fp32 accumulate",
        "data": "synthetic (random-init weights, N(0,1) fp16 X)",
        "config": config,
        "tflops": round(flops / t_step / 1e12, 3),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": round(achieved / peaks["hbm_gbs"], 4), "traffic": traffic,
                     "traffic_unit": "bytes per step (DRAM read + write, ncu)", "traffic_detail": traffic_note,
                     "peak_source": peaks["source"],
                     "kernel": "w6a16_tcgen05_kernel<16> (all 4 launches of the step, timed region)",
                     "per_launch_serialised": res["per_layer"]},
        "cublas_fp16": dict(res["cublas"], speedup_vs_cublas=round(res["cublas"]["ms_per_step"] / (t_step * 1e3), 3)),
        "e2e": res["e2e"],
        "gpu_launches": res["gpu_launches"],
        "clocks": res["clocks"],
        "extras": extras,
    }
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(layers, m)
    print(json.dumps(line), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
