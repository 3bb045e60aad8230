#!/usr/bin/env python
"""bench.py -- W4A16 GEMM throughput on B200 vs roofline (BASELINE.json metric).

A *step* is one pass of the hot path over the workload's GEMM list; for the default workload
(BASELINE.json configs[1], Llama-2-7B attention projection N = K = 4096, g128) that is the
M sweep 1, 2, 4, ..., 256: nine quick_w4a16_gemm launches on synthetic AWQ weights.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl quick|reference] [--workload W]

Timing: weights are packed offline once (host, C++), then R device copies of the
blob rotate launch by launch so every launch streams its weights from HBM (R copies > 2.5 x L2),
never from L2.  The K timed steps run as CUDA-graph replays, M-major in blocks of C steps (graph
per M point holding C launches), with CUDA events on the launching stream between graph
replays, so the per-M average launch duration is measured over the whole timed region.
`value` = whole-job TFLOP/s (2 M N K per GEMM, all ranks) over the max-over-ranks device time.
`e2e`  = same metric through the C-ABI with HOST buffers: every step copies X from pinned host
memory and Y back to pinned host memory inside the timed region (weights stay resident).
N > 1: tensor parallel, weights column-sharded along N (multiples of 128), each rank runs the
GEMM on its shard, then NCCL all-gather + quick_gather_columns materialise Y (strong scaling).
"""
import argparse
import json
import os
import statistics
import sys
import threading
import time

import numpy as np

# debug/ablation only: extra internal launch flags OR-ed into the timed launches (e.g. 0x80000 =
# automatic plan without CTA pairs); 0 for every reported number
EXTRA_FLAGS = int(os.environ.get("QUICK_BENCH_EXTRA_FLAGS", "0"), 0)

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import synth  # noqa: E402  (seeded random bits only)

WORKLOADS = {
    # name: (BASELINE.json config index, list of (N, K) shapes, M points, G)
    "llama2_7b_attn": (1, [(4096, 4096)], [1, 2, 4, 8, 16, 32, 64, 128, 256], 128),
    "llama2_13b_mlp": (2, [(13824, 5120), (5120, 13824)], [1, 2, 4, 8, 16, 32, 64, 128, 256, 512], 128),
    "llama2_70b_mlp": (3, [(28672, 8192)], [1, 16, 64, 128, 256, 512, 1024], 128),
    "tiny": (0, [(256, 512)], [8], 128),
    # BASELINE.json configs[4]: one Mistral-7B decoder layer's linear stack (QKV, O, gate_up, down);
    # tokens/s = M / (32 layers x the 4 GEMMs' time); attention, norms and SiLU are not on the path
    "mistral7b_stack": (4, [(6144, 4096), (4096, 4096), (28672, 4096), (4096, 14336)], [1, 16, 64, 256], 128),
}
METRIC = "W4A16 GEMM TFLOP/s & HBM GB/s vs roofline, M=1–1024, 1/2/4/8 B200"
BLOCK_C = 32  # steps per graph replay (M-major): PDL overlaps consecutive launches inside a graph


def algo_bytes(M, N, K, G):
    """int4 weights + fp16 scales + 4-bit zeros + X once + Y once."""
    return K * N // 2 + (K // G) * N * 5 // 2 + 2 * M * K + 2 * M * N


def algo_flops(M, N, K):
    return 2 * M * N * K


def load_peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            p = json.load(f)
        return {"hbm_gbs": float(p["hbm_gbs"]), "tflops": float(p["bf16_tflops"]),
                "tflops_sustained": float(p.get("bf16_tflops_sustained", p["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json; fp16 dense = bf16 dense x 1.0 nominal ratio)"}
    except Exception:
        return {"hbm_gbs": 6650.0, "tflops": 1590.0, "tflops_sustained": 1400.0,
                "source": "fallback (B200_PROFILING.md)"}


def load_traffic():
    """ncu dram bytes per launch (committed under profiles/), keyed 'workload:N:K:M'."""
    path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return {}


# ------------------------------------------------------------------------------------------ clocks
class ClockSampler:
    """NVML sampling of SM clock and throttle reasons during the timed region (~1 ms period)."""

    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown",
               0x4: "sw_power_cap", 0x80: "hw_power_brake_slowdown", 0x2: "applications_clocks_setting"}

    def __init__(self, index):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None
        self._stop = threading.Event()

    def _run(self):
        nv = self.nv
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                fn = getattr(nv, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                    nv.nvmlDeviceGetCurrentClocksThrottleReasons
                r = fn(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.001)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


# ------------------------------------------------------------------------------------------ GPU arm
def run_quick(args, rank, world, dist):
    import torch
    from paper_2402_10076_b200 import quick

    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)))
    torch.cuda.set_device(dev)
    cfg_idx, shapes, Ms, G = WORKLOADS[args.workload]
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20)

    # ---- problem: per shape, synthetic AWQ weights, column shard for this rank, offline pack
    gemms = []   # one entry per (shape, M): dict
    shard_info = []
    blobs = []
    pack_s = 0.0
    for si, (N, K) in enumerate(shapes):
        assert N % (128 * world) == 0, "column shard must be a multiple of 128"
        Nr = N // world
        qw = synth.make_qweight(si, K, N)
        sc = synth.make_scales(si, K, N, G)
        zr = synth.make_zeros(si, K, N, G)
        c0 = rank * Nr
        t0 = time.perf_counter()
        blob = quick.quick_pack_weights(qw[:, c0 // 8:(c0 + Nr) // 8], sc[:, c0:c0 + Nr], zr[:, c0 // 8:(c0 + Nr) // 8], G)
        pack_s += time.perf_counter() - t0
        blobs.append(blob)
        shard_info.append((N, K, Nr))
    blob_bytes = max(b.size for b in blobs)
    per_step_launches = len(shapes) * len(Ms)
    # weight copies: reuse distance >= 2.5 x L2 and a multiple of the launches per graph block
    # slot of launch c of GEMM gi inside a block = (gi * C + c) % R; R divides the launches per
    # block so the reuse distance of every slot is exactly R launches (> 2.5 x L2 of weights)
    launches_per_rep = per_step_launches * BLOCK_C
    R_min = max(1, int(np.ceil(2.5 * l2 / blob_bytes)))
    l2_cold = R_min <= launches_per_rep
    R = min(d for d in range(R_min, launches_per_rep + 1) if launches_per_rep % d == 0) if l2_cold \
        else launches_per_rep
    wcopies = {}
    for si, blob in enumerate(blobs):
        base = torch.from_numpy(blob).to(dev)
        wcopies[si] = [base] + [base.clone() for _ in range(R - 1)]
    # activations: per (shape, M) R copies too (cold), outputs per (shape, M)
    for si, (N, K, Nr) in enumerate(shard_info):
        for mi, M in enumerate(Ms):
            x_host = synth.make_x(1000 + M, M, K)
            xs = [torch.from_numpy(x_host.view(np.int16)).view(torch.float16).to(dev) for _ in range(min(R, 8))]
            y = torch.empty((M, Nr), device=dev, dtype=torch.float16)
            plan = quick.quick_gemm_plan(M, Nr, K, G)
            gemms.append(dict(si=si, M=M, N=N, K=K, Nr=Nr, xs=xs, y=y, plan=plan, x_host=x_host,
                              gathered=torch.empty((world, M, Nr), device=dev, dtype=torch.float16) if world > 1 else None,
                              yfull=torch.empty((M, N), device=dev, dtype=torch.float16) if world > 1 else None))

    stream = torch.cuda.Stream(dev)        # graph capture needs a non-default stream
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream

    # back-to-back GEMMs of a decode step: programmatic dependent launch lets each launch's
    # prologue and weight prefetch overlap the previous kernel's tail (X / Y stay ordered)
    def launch(g, slot):
        x = g["xs"][slot % len(g["xs"])]
        quick.quick_w4a16_gemm_raw(x.data_ptr(), wcopies[g["si"]][slot].data_ptr(), g["M"], g["Nr"], g["K"], G,
                                   g["y"].data_ptr(), sh, flags=quick.QUICK_FLAG_PDL | EXTRA_FLAGS)

    for g in gemms:   # eager first: allocates the stream-K workspace outside graph capture
        launch(g, 0)
    torch.cuda.synchronize()

    # graph per (gemm index, block size C): C launches of that GEMM with rotating weight slots;
    # launch index inside a rep = gi * C + c -> slot (gi * C + c) % R  (R divides gi-count * C)
    def build_graphs(C):
        graphs = []
        for gi, g in enumerate(gemms):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                for c in range(C):
                    launch(g, (gi * C + c) % R)
            graphs.append(gr)
        return graphs

    def collective(g):
        # column-parallel TP: all-gather the per-rank [M][Nr] slices, then permute to [M][N]
        dist.all_gather_into_tensor(g["gathered"].view(-1), g["y"].view(-1))
        quick.quick_gather_columns(g["gathered"], world, g["M"], g["Nr"], dst=g["yfull"])

    K_steps, W = args.steps, args.warmup
    graphs_full = build_graphs(BLOCK_C)
    rem = K_steps % BLOCK_C
    graphs_rem = build_graphs(rem) if rem else []
    torch.cuda.synchronize()
    for gr in graphs_full + graphs_rem:   # upload / first-touch every graph before warm-up
        gr.replay()
    torch.cuda.synchronize()

    def run_steps(nsteps, record=None):
        """nsteps steps as graph replays, M-major in blocks of BLOCK_C (+ remainder block)."""
        blocks = [BLOCK_C] * (nsteps // BLOCK_C) + ([nsteps % BLOCK_C] if nsteps % BLOCK_C else [])
        for C in blocks:
            grs = graphs_full if C == BLOCK_C else (graphs_rem if C == rem else build_graphs(C))
            for gi, gr in enumerate(grs):
                if record is not None:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(stream)
                    record.append((gi, C, ev))
                gr.replay()
                if world > 1:
                    for _ in range(C):
                        collective(gemms[gi])
        if record is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            record.append((None, 0, ev))

    run_steps(W)     # W untimed warm-up steps
    torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    rec = []
    sampler = ClockSampler(dev.index)
    with sampler:
        t_start = torch.cuda.Event(enable_timing=True)
        t_end = torch.cuda.Event(enable_timing=True)
        t_start.record(stream)
        run_steps(K_steps, rec)
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = t_start.elapsed_time(t_end)
    if dist is not None:
        t = torch.tensor([elapsed_ms], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        elapsed_ms = float(t.item())

    # per-GEMM average launch duration over the timed region (events between graph replays)
    per_gemm_ms = [0.0] * len(gemms)
    per_gemm_n = [0] * len(gemms)
    for (gi, C, ev), (_, _, ev_next) in zip(rec[:-1], rec[1:]):
        per_gemm_ms[gi] += ev.elapsed_time(ev_next)
        per_gemm_n[gi] += C

    peaks = load_peaks()
    ridge = peaks["tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    traffic = load_traffic()
    step_flops = sum(algo_flops(g["M"], g["N"], g["K"]) for g in gemms)
    step_bytes_rank = sum(algo_bytes(g["M"], g["Nr"], g["K"], G) for g in gemms)
    sweep = []
    for gi, g in enumerate(gemms):
        us = 1e3 * per_gemm_ms[gi] / max(1, per_gemm_n[gi])
        fl = algo_flops(g["M"], g["Nr"], g["K"])
        by = algo_bytes(g["M"], g["Nr"], g["K"], G)
        tfl = fl / (us * 1e-6) / 1e12
        gbs = by / (us * 1e-6) / 1e9
        sweep.append({"M": g["M"], "N": g["Nr"], "K": g["K"], "us": round(us, 3), "tflops": round(tfl, 2),
                      "gbs": round(gbs, 1), "frac_hbm": round(gbs / peaks["hbm_gbs"], 4),
                      "frac_tensor": round(tfl / peaks["tflops"], 4),
                      "bound": "tensor" if fl / by >= ridge else "hbm",
                      "tile_n": g["plan"]["tile_n"], "split_k": g["plan"]["split_k"],
                      "cta_pair": g["plan"].get("pair", False),
                      "ctas": g["plan"]["num_ctas"]})
    layer_stack = None
    if args.workload == "mistral7b_stack":
        # per batch size: the 4 GEMMs of one layer back to back, x 32 layers
        layer_stack = []
        for M in Ms:
            us_layer = sum(e["us"] for e in sweep if e["M"] == M)
            layer_stack.append({"M": M, "us_per_layer": round(us_layer, 3),
                                "tokens_per_s": round(M / (32 * us_layer * 1e-6), 1)})
    dom = max(range(len(gemms)), key=lambda i: per_gemm_ms[i])
    d = sweep[dom]
    if d["bound"] == "tensor":
        roof = {"bound": "tensor", "achieved": d["tflops"], "peak": peaks["tflops"], "unit": "TFLOP/s",
                "frac": round(d["tflops"] / peaks["tflops"], 4)}
    else:
        roof = {"bound": "hbm", "achieved": d["gbs"], "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(d["gbs"] / peaks["hbm_gbs"], 4)}
    tkey = f"{args.workload}:{d['N']}:{d['K']}:{d['M']}"
    roof["traffic"] = traffic.get(tkey)
    roof["kernel"] = (f"quick_w4a16_tc_kernel<{d['tile_n']}{', cta_group::2 pair' if d.get('cta_pair') else ''}> "
                      f"M={d['M']} N={d['N']} K={d['K']} split_k={d['split_k']}")
    roof["algorithmic_per_launch"] = algo_bytes(d["M"], d["N"], d["K"], G) if d["bound"] == "hbm" else \
        algo_flops(d["M"], d["N"], d["K"])
    roof["peak_source"] = peaks["source"]
    roof["share_of_step"] = round(per_gemm_ms[dom] / sum(per_gemm_ms), 4)

    # ---- e2e: through the C-ABI with host buffers (pinned), copies inside the timed region
    e2e = run_e2e(args, gemms, wcopies, R, G, stream, dist, world, quick, collective)

    value = K_steps * step_flops / (elapsed_ms * 1e-3) / 1e12
    gbs_all = K_steps * step_bytes_rank * world / (elapsed_ms * 1e-3) / 1e9
    res = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": K_steps,
        "warmup": W, "ms_per_step": round(elapsed_ms / K_steps, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (SplitMix64 AWQ int4 weights, U[-1,1] fp16 X)",
        "config": {"workload": args.workload, "baseline_config": cfg_idx,
                   "shapes_NxK": [[n, k] for n, k in shapes], "M": Ms, "group_size": G,
                   "gemms_per_step": per_step_launches,
                   "parallelism": f"tp{world} column-sharded N, NCCL all-gather" if world > 1 else "single GPU",
                   "l2": (f"rotating {R} weight copies ({R * blob_bytes / 2**20:.0f} MiB) > L2 {l2 / 2**20:.0f} MiB; "
                          "every launch reads its weights from HBM") if l2_cold else
                         f"weights L2-resident ({R} copies of {blob_bytes} B < 2.5 x L2)",
                   "timing": f"CUDA-graph replays of {BLOCK_C} launches per M point (PDL between consecutive launches), M-major; events between replays",
                   "launch": "quick_w4a16_gemm_ex with QUICK_FLAG_PDL (programmatic dependent launch), automatic plan"},
        "hbm_gbs_aggregate": round(gbs_all, 1),
        "gpu_launches": K_steps * per_step_launches * (2 if world > 1 else 1),
        "roofline": roof,
        "sweep": sweep,
        **({"layer_stack_32_layers": layer_stack} if layer_stack else {}),
        "e2e": e2e,
        "pack": {"host_seconds": round(pack_s, 4), "bytes": int(sum(b.size for b in blobs))},
        "clocks": sampler.summary(),
    }
    return res


def run_e2e(args, gemms, wcopies, R, G, stream, dist, world, quick, collective):
    import torch
    steps = max(3, min(args.steps, 200))
    xh = [torch.from_numpy(g["x_host"].view(np.int16)).view(torch.float16).pin_memory() for g in gemms]
    yh = [torch.empty(g["yfull"].shape if world > 1 else g["y"].shape, dtype=torch.float16).pin_memory() for g in gemms]
    xd = [g["xs"][0] for g in gemms]
    sh = stream.cuda_stream

    pipelined = world == 1
    if pipelined:
        # copies overlap the GEMMs, as a serving loop would run them: X uploads on one copy
        # stream, Y downloads on another, the GEMMs on `stream`; per-GEMM buffers and events
        # order each GEMM after its upload and each download after its GEMM, and an upload /
        # GEMM waits for the previous step's use of its buffer
        s_h2d, s_d2h = torch.cuda.Stream(stream.device), torch.cuda.Stream(stream.device)
        ev = {k: [torch.cuda.Event() for _ in gemms] for k in ("h2d", "comp", "d2h")}
        started = [False] * len(gemms)

    def step(i):
        for gi, g in enumerate(gemms):
            slot = (i * len(gemms) + gi) % R
            if not pipelined:
                xd[gi].copy_(xh[gi], non_blocking=True)
                quick.quick_w4a16_gemm_raw(xd[gi].data_ptr(), wcopies[g["si"]][slot].data_ptr(), g["M"], g["Nr"],
                                           g["K"], G, g["y"].data_ptr(), sh)
                if world > 1:
                    collective(g)
                    yh[gi].copy_(g["yfull"], non_blocking=True)
                else:
                    yh[gi].copy_(g["y"], non_blocking=True)
                continue
            with torch.cuda.stream(s_h2d):
                if started[gi]:
                    s_h2d.wait_event(ev["comp"][gi])      # the previous GEMM on xd[gi] is done
                xd[gi].copy_(xh[gi], non_blocking=True)
                ev["h2d"][gi].record(s_h2d)
            stream.wait_event(ev["h2d"][gi])
            if started[gi]:
                stream.wait_event(ev["d2h"][gi])          # y[gi] has been read back
            quick.quick_w4a16_gemm_raw(xd[gi].data_ptr(), wcopies[g["si"]][slot].data_ptr(), g["M"], g["Nr"],
                                       g["K"], G, g["y"].data_ptr(), sh)
            ev["comp"][gi].record(stream)
            with torch.cuda.stream(s_d2h):
                s_d2h.wait_event(ev["comp"][gi])
                yh[gi].copy_(g["y"], non_blocking=True)
                ev["d2h"][gi].record(s_d2h)
            started[gi] = True

    for i in range(3):
        step(i)
    torch.cuda.synchronize()
    graph = None
    if pipelined:
        # one step = one CUDA-graph replay: the 9 uploads, GEMMs (C-ABI calls, captured) and
        # read-backs with their cross-stream event edges, forked from and joined to `stream`
        # (replays on `stream` are ordered, so buffers are reused safely across steps)
        graph = torch.cuda.CUDAGraph()
        with torch.cuda.graph(graph, stream=stream):
            fork = torch.cuda.Event()
            fork.record(stream)
            s_h2d.wait_event(fork)
            s_d2h.wait_event(fork)
            started[:] = [False] * len(gemms)
            step(0)
            for gi in range(len(gemms)):
                stream.wait_event(ev["d2h"][gi])
            stream.wait_event(ev["h2d"][len(gemms) - 1])
        graph.replay()
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record(stream)
    for i in range(steps):
        if graph is not None:
            graph.replay()
        else:
            step(i)
    b.record(stream)
    torch.cuda.synchronize()
    ms = a.elapsed_time(b)
    if dist is not None:
        t = torch.tensor([ms], device=stream.device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    flops = sum(algo_flops(g["M"], g["N"], g["K"]) for g in gemms)
    return {"value": round(steps * flops / (ms * 1e-3) / 1e12, 4), "unit": "TFLOP/s",
            "h2d_bytes_per_step": int(sum(2 * g["M"] * g["K"] for g in gemms)),
            "d2h_bytes_per_step": int(sum(2 * g["M"] * g["N"] for g in gemms)),
            "steps": steps, "ms_per_step": round(ms / steps, 4),
            "path": ("C-ABI quick_w4a16_gemm per GEMM, pinned H2D X + D2H Y each step"
                     + ("; one CUDA-graph replay per step holding the uploads, the captured C-ABI GEMM calls and "
                        "the read-backs on three streams with event dependencies (copies overlap GEMMs)"
                        if world == 1 else ""))}


# ------------------------------------------------------------------------------------------ CPU arm
def oracle_step_sample(workload, budget_s):
    """Time the oracle (as it stands) on a bounded sample of one step of the workload:
    every GEMM of the step restricted to the first n_s output columns (n_s % 8 == 0)."""
    import oracle  # bench.py's cpu_baseline / reference leg is allowed to call the oracle
    _, shapes, Ms, G = WORKLOADS[workload]
    probs = []
    for si, (N, K) in enumerate(shapes):
        qw = synth.make_qweight(si, K, N)
        sc = synth.make_scales(si, K, N, G)
        zr = synth.make_zeros(si, K, N, G)
        probs.append((N, K, qw, sc, zr))

    xs = {(K, M): synth.make_x(1000 + M, M, K) for (N, K, *_r) in probs for M in Ms}

    def one(ns):
        fl = 0
        t0 = time.perf_counter()
        for (N, K, qw, sc, zr) in probs:
            n = min(ns, N)
            for M in Ms:
                oracle.w4a16_reference(xs[(K, M)], qw[:, :n // 8], sc[:, :n], zr[:, :n // 8], G)
                fl += 2 * M * n * K
        return time.perf_counter() - t0, fl

    N_max = max(N for N, *_ in probs)
    ns, t = 64, 0.0
    while True:                                           # calibrate: grow the sample geometrically
        t, _ = one(ns)
        if t >= budget_s / 4 or ns >= N_max:
            break
        ns *= 2
    ns = int(max(8, min(N_max, ns * budget_s / max(t, 1e-6))) // 8 * 8)
    return ns, one


def cpu_threads():
    try:
        from threadpoolctl import threadpool_info
        info = threadpool_info()
        return max((i.get("num_threads", 1) for i in info), default=1)
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(workload, budget_s=15.0):
    ns, one = oracle_step_sample(workload, budget_s)
    t, fl = one(ns)
    return {"value": round(fl / t / 1e12, 6), "unit": "TFLOP/s", "cores": cpu_threads(), "kind": "oracle",
            "sample": f"one step of {workload} with every GEMM restricted to the first {ns} output columns "
                      f"(oracle O1-O3 in numpy fp64, dequant per call); {t:.1f} s",
            "host_cpus": os.cpu_count()}


def run_reference(args):
    _, shapes, Ms, G = WORKLOADS[args.workload]
    per_step_budget = max(0.05, 90.0 / max(1, args.steps + args.warmup))
    ns, one = oracle_step_sample(args.workload, per_step_budget)
    for _ in range(args.warmup):
        one(ns)
    tot_t, tot_f = 0.0, 0
    for _ in range(args.steps):
        t, f = one(ns)
        tot_t += t
        tot_f += f
    v = tot_f / tot_t / 1e12
    sample = f"each step = one step of {args.workload} restricted to the first {ns} output columns"
    return {"metric": METRIC, "value": round(v, 6), "unit": "TFLOP/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(1e3 * tot_t / args.steps, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "impl": "reference",
            "config": {"workload": args.workload, "group_size": G, "M": Ms,
                       "shapes_NxK": [[n, k] for n, k in shapes], "columns_per_gemm": ns},
            "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "kind": "oracle", "cores": cpu_threads(),
                             "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------------------------------ main
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=800)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["quick", "reference"], default="quick")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default="llama2_7b_attn")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    args = ap.parse_args()
    assert args.warmup >= 3 and args.steps >= 1

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))

    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
        tdist.init_process_group("nccl")
        dist = tdist
    res = run_quick(args, rank, world, dist)
    if rank == 0:
        if world == 1 and not args.no_cpu_baseline:
            res["cpu_baseline"] = cpu_baseline(args.workload, args.cpu_budget)
        print(json.dumps(res), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
