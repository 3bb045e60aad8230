#!/usr/bin/env python
"""bench.py -- W4A16 GEMM throughput on B200 vs roofline (BASELINE.json metric).

A *step* is one pass of the hot path over the workload's GEMM list.  The default workload is the
one the metric ("M=1-1024, 1/2/4/8 B200") is quoted on, BASELINE.json configs[3]: the Llama-2-70B
MLP pair, the up-projection 28672x8192 (K=8192 -> N=28672, column-parallel) and the
down-projection 8192x28672 (K=28672 -> N=8192, row-parallel), g128, each at
M = 1, 4, 16, 64, 128, 256, 512, 1024: sixteen quick_w4a16_gemm_ex launches on synthetic AWQ
weights.  Other configs: --workload llama2_7b_attn (configs[1]), llama2_13b_mlp (configs[2]),
mistral7b_stack (configs[4]), tiny (configs[0]), paper_fig7 (the paper's 8192x8192 sweep).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl quick|reference] [--workload W]

--gpus N > 1 without a torchrun environment re-launches itself under torch.distributed.run with
N ranks (127.0.0.1); under torchrun WORLD_SIZE must equal N.

Timing: weights are packed offline once (host, C++), then R device copies of each
blob rotate launch by launch so every launch streams its weights from HBM (R copies > 2.5 x L2).
The K timed steps run as CUDA-graph replays, GEMM-point-major in blocks of C steps, with CUDA events
on the launching stream between replays, so each point's mean launch duration is measured over the
whole timed region.  `value` = whole-job TFLOP/s (2 M N K per GEMM, all ranks) over the
max-over-ranks device time.  Launches use QUICK_FLAG_PDL and a caller-owned stream-K workspace.
`e2e` = the same metric through the C-ABI with HOST buffers: every step copies X from pinned host
memory and Y back to pinned host memory inside the timed region (weights stay resident).
N > 1: tensor parallel (strong scaling); column-parallel GEMMs shard N (multiples of 128) and
all-gather Y (NCCL) + quick_gather_columns; row-parallel GEMMs shard K (group-aligned), write fp32
partials, all-reduce them in fp32 (NCCL) + quick_f32_to_f16.  GEMM-only and GEMM+collective
times are reported separately.
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
    # name: (BASELINE.json config index, list of (N, K, tp kind) shapes, M points, G);
    # tp kind "col" = column-parallel (N sharded), "row" = row-parallel (K sharded, fp32 all-reduce)
    "llama2_70b_mlp": (3, [(28672, 8192, "col"), (8192, 28672, "row")], [1, 4, 16, 64, 128, 256, 512, 1024], 128),
    "llama2_7b_attn": (1, [(4096, 4096, "col")], [1, 2, 4, 8, 16, 32, 64, 128, 256], 128),
    "llama2_13b_mlp": (2, [(13824, 5120, "col"), (5120, 13824, "row")], [1, 2, 4, 8, 16, 32, 64, 128, 256, 512],
                       128),
    "tiny": (0, [(256, 512, "col")], [8], 128),
    # BASELINE.json configs[4]: one Mistral-7B decoder layer's linear stack (QKV, O, gate_up, down) in the
    # Megatron split: QKV column-parallel by head group and the fused gate||up GEMM with its SiLU*mul
    # epilogue ("silu": quick_pack_gate_up + QUICK_FLAG_SILU_MUL) column-parallel (their sharded outputs
    # feed the next GEMM, so no gather), O and down row-parallel (fp32 all-reduce); tokens/s = M / (32
    # layers x the 4 GEMMs' time); attention and norms are not on the path
    "mistral7b_stack": (4, [(6144, 4096, "colx"), (4096, 4096, "row"), (28672, 4096, "silu"), (4096, 14336, "row")],
                        [1, 16, 64, 256], 128),
    # the paper's kernel benchmark shape (Fig. 7): 8192 x 8192, batch 64 .. 512 (context)
    "paper_fig7": (None, [(8192, 8192, "col")], [1, 16, 64, 128, 256, 512], 128),
}
DEFAULT_WORKLOAD = "llama2_70b_mlp"
METRIC = "W4A16 GEMM TFLOP/s & HBM GB/s vs roofline, M=1–1024, 1/2/4/8 B200"
BLOCK_C = 32  # steps per graph replay (M-major): PDL overlaps consecutive launches inside a graph


def algo_bytes(M, N, K, G, n_out=None):
    """int4 weights + fp16 scales + 4-bit zeros + X once + Y once (n_out columns of Y:
    N, or N/2 for the fused gate||up SiLU epilogue)."""
    return K * N // 2 + (K // G) * N * 5 // 2 + 2 * M * K + 2 * M * (N if n_out is None else n_out)


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
def tp_desc(kind, peer):
    if kind == "col":
        return "column-parallel, all-gather fused into the GEMM epilogue (peer memory)" if peer else \
            "column-parallel + NCCL all-gather"
    if kind == "colx":
        return "column-parallel (output stays sharded)"
    if kind == "silu":
        return "fused gate||up + SiLU*mul, column-parallel (output stays sharded)"
    return "row-parallel + peer-memory fp32 all-reduce" if peer else "row-parallel + NCCL fp32 all-reduce"


def plan_key(plan):
    """Kernel identity of a launch: the template instantiation and grid family it runs."""
    sched = "stream-K" if plan["split_k"] == 0 else f"split{plan['split_k']}"
    return f"tile{plan['tile_n']}{'-pair' if plan['pair'] else ''}-{sched}"


def run_quick(args, rank, world, dist):
    import torch
    from paper_2402_10076_b200 import quick, tp

    # (--dist-backend gloo, a test mode: several ranks may share one GPU)
    dev = torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
    torch.cuda.set_device(dev)
    cfg_idx, shapes, Ms, G = WORKLOADS[args.workload]
    props = torch.cuda.get_device_properties(dev)
    l2 = int(getattr(props, "L2_cache_size", 126 * 2**20) or 126 * 2**20)

    # ---- problem: per shape, synthetic AWQ weights, this rank's shard, offline pack (host, C++)
    layers, pack_s = [], 0.0
    for si, (N, K, kind) in enumerate(shapes):
        qw, sc, zr = synth.make_qweight(si, K, N), synth.make_scales(si, K, N, G), synth.make_zeros(si, K, N, G)
        if kind == "silu":
            # fused gate||up: columns [0, N/2) = gate, [N/2, N) = up; rank r keeps the same I/P slice of both
            I = N // 2
            gate = (qw[:, :I // 8], sc[:, :I], zr[:, :I // 8])
            up = (qw[:, I // 8:], sc[:, I:], zr[:, I // 8:])
            gate, up = tp.shard_gate_up(gate, up, rank, world)
            Nl, Kl = N // world, K
            t0 = time.perf_counter()
            blob = quick.quick_pack_gate_up(gate, up, G)
            pack_s += time.perf_counter() - t0
            layers.append(dict(si=si, N=N, K=K, kind=kind, Nl=Nl, Kl=Kl, n_out=Nl // 2, blob=blob))
            continue
        if world > 1 and kind in ("col", "colx"):
            qw, sc, zr = tp.shard_awq_columns(qw, sc, zr, rank, world)
            Nl, Kl = N // world, K
        elif world > 1:
            qw, sc, zr = tp.shard_awq_rows(qw, sc, zr, G, rank, world)
            Nl, Kl = N, K // world
        else:
            Nl, Kl = N, K
        t0 = time.perf_counter()
        blob = quick.quick_pack_weights(qw, sc, zr, G)
        pack_s += time.perf_counter() - t0
        layers.append(dict(si=si, N=N, K=K, kind=kind, Nl=Nl, Kl=Kl, n_out=Nl, blob=blob))
    blob_bytes = max(l_["blob"].size for l_ in layers)
    launches_per_rep = len(layers) * len(Ms) * BLOCK_C
    # weight copies: reuse distance >= 2.5 x L2 (slot of launch c of point gi = (gi * C + c) % R, R
    # divides the launches per block, so every slot is reused exactly R launches later)
    R_min = max(1, int(np.ceil(2.5 * l2 / blob_bytes)))
    l2_cold = R_min <= launches_per_rep
    R = min(d for d in range(R_min, launches_per_rep + 1) if launches_per_rep % d == 0) if l2_cold \
        else launches_per_rep
    wcopies = {}
    for l_ in layers:
        base = torch.from_numpy(l_["blob"]).to(dev)
        wcopies[l_["si"]] = [base] + [base.clone() for _ in range(R - 1)]
    ws = quick.workspace_for([(M, l_["Nl"], l_["Kl"]) for l_ in layers for M in Ms], G, dev)
    ws_ptr, ws_bytes = ws.data_ptr(), ws.numel()

    gemms = []   # one entry per (shape, M) point
    for l_ in layers:
        for M in Ms:
            x_host = synth.make_x(1000 + M, M, l_["K"])
            if world > 1 and l_["kind"] == "row":
                k0, k1 = tp.row_shard_bounds(l_["K"], G, world, rank)
                x_host = np.ascontiguousarray(x_host[:, k0:k1])
            xs = [torch.from_numpy(x_host.view(np.int16)).view(torch.float16).to(dev) for _ in range(min(R, 8))]
            row_partial = world > 1 and l_["kind"] == "row"
            y = torch.empty((M, l_["n_out"]), device=dev, dtype=torch.float32 if row_partial else torch.float16)
            g = dict(l_, M=M, xs=xs, y=y, x_host=x_host,
                     plan=quick.quick_gemm_plan(M, l_["Nl"], l_["Kl"], G, workspace_bytes=ws_bytes,
                                                flags=quick.QUICK_FLAG_SILU_MUL if l_["kind"] == "silu" else 0))
            if world > 1 and l_["kind"] == "col":
                g["gathered"] = torch.empty((world, M, l_["Nl"]), device=dev, dtype=torch.float16)
                g["yfull"] = torch.empty((M, l_["N"]), device=dev, dtype=torch.float16)
            if row_partial:
                g["yfull"] = torch.empty((M, l_["N"]), device=dev, dtype=torch.float16)
            gemms.append(g)

    stream = torch.cuda.Stream(dev)        # graph capture needs a non-default stream
    torch.cuda.set_stream(stream)
    sh = stream.cuda_stream

    # back-to-back GEMMs of a decode step: programmatic dependent launch lets each launch's
    # prologue and weight prefetch overlap the previous kernel's tail (X / Y stay ordered)
    def launch(g, slot):
        x = g["xs"][slot % len(g["xs"])]
        fl = quick.QUICK_FLAG_PDL | EXTRA_FLAGS | (quick.QUICK_FLAG_OUT_F32 if g["y"].dtype == torch.float32 else 0) \
            | (quick.QUICK_FLAG_SILU_MUL if g["kind"] == "silu" else 0)
        quick.quick_w4a16_gemm_raw(x.data_ptr(), wcopies[g["si"]][slot].data_ptr(), g["M"], g["Nl"], g["Kl"], G,
                                   g["y"].data_ptr(), sh, flags=fl, ws_ptr=ws_ptr, ws_bytes=ws_bytes,
                                   ldy=g["n_out"])

    peer = world > 1 and args.comm == "peer"
    if peer:
        # collective-fused TP over peer memory: symmetric buffers (CUDA IPC, handles
        # exchanged over the NCCL group), the column-parallel all-gather fused into the GEMM epilogue,
        # the row-parallel fp32 all-reduce done by our own peer-memory kernel; two Y buffers per point
        comm = tp.PeerComm()
        for g in gemms:
            if g["kind"] == "col":
                g["ypeer"] = [comm.buffer(g["M"] * g["N"] * 2) for _ in range(2)]
            elif g["kind"] == "row":
                g["ppeer"] = comm.buffer(g["M"] * g["N"] * 4)
                g["ypeer"] = [comm.buffer(g["M"] * g["N"] * 2) for _ in range(2)]
            g["turn"] = 0

    def launch_peer(g, slot):
        x = g["xs"][slot % len(g["xs"])]
        w = wcopies[g["si"]][slot]
        yp = g["ypeer"][g["turn"]]
        g["turn"] ^= 1
        if g["kind"] == "col":
            quick.quick_tp_column_gemm(x, w, g["Nl"], g["Kl"], G, yp, g["N"], comm.flags, rank,
                                       flags=quick.QUICK_FLAG_PDL | EXTRA_FLAGS, workspace=ws)
        else:
            quick.quick_tp_row_gemm(x, w, g["N"], g["Kl"], G, g["ppeer"], yp, g["N"], comm.flags, rank,
                                    flags=quick.QUICK_FLAG_PDL | EXTRA_FLAGS, workspace=ws)

    def collective(g):
        if world == 1 or g["kind"] in ("colx", "silu"):
            return          # colx / silu: the sharded output feeds the next (row-parallel) GEMM, no gather
        if g["kind"] == "col":   # all-gather the per-rank [M][Nr] slices, then permute to [M][N]
            dist.all_gather_into_tensor(g["gathered"].view(-1), g["y"].view(-1))
            quick.quick_gather_columns(g["gathered"], world, g["M"], g["Nl"], dst=g["yfull"])
        else:                    # row: fp32 all-reduce of the partials, then cast
            dist.all_reduce(g["y"], op=dist.ReduceOp.SUM)
            quick.quick_f32_to_f16(g["y"], dst=g["yfull"])

    for g in gemms:
        if peer and g["kind"] in ("col", "row"):
            launch_peer(g, 0)
        else:
            launch(g, 0)
            collective(g)
    torch.cuda.synchronize()

    # graph per GEMM point holding C launches (+ their collectives when `with_coll`; with --comm peer
    # the collective-fused TP calls replace both)
    def build_graphs(C, with_coll):
        graphs = []
        for gi, g in enumerate(gemms):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=stream):
                for c in range(C):
                    if with_coll and peer and g["kind"] in ("col", "row"):
                        launch_peer(g, (gi * C + c) % R)
                        continue
                    launch(g, (gi * C + c) % R)
                    if with_coll:
                        collective(g)
            graphs.append(gr)
        return graphs

    K_steps, W = args.steps, args.warmup
    coll_in_graph = world > 1 and (peer or args.dist_backend == "nccl")   # gloo collectives cannot be captured
    try:
        graphs_full = build_graphs(BLOCK_C, coll_in_graph)
    except Exception:        # a NCCL build that cannot be captured: collectives run eagerly
        torch.cuda.synchronize()
        coll_in_graph = False
        graphs_full = build_graphs(BLOCK_C, False)
    rem = K_steps % BLOCK_C
    graphs_rem = build_graphs(rem, coll_in_graph) if rem else []
    torch.cuda.synchronize()
    for gr in graphs_full + graphs_rem:   # upload / first-touch every graph before warm-up
        gr.replay()
    torch.cuda.synchronize()

    def run_steps(nsteps, grs_full, grs_rem, eager_coll, record=None):
        """nsteps steps as graph replays, point-major in blocks of BLOCK_C (+ remainder block)."""
        blocks = [BLOCK_C] * (nsteps // BLOCK_C) + ([nsteps % BLOCK_C] if nsteps % BLOCK_C else [])
        for C in blocks:
            grs = grs_full if C == BLOCK_C else grs_rem
            for gi, gr in enumerate(grs):
                if record is not None:
                    ev = torch.cuda.Event(enable_timing=True)
                    ev.record(stream)
                    record.append((gi, C, ev))
                gr.replay()
                if eager_coll:
                    for _ in range(C):
                        collective(gemms[gi])
        if record is not None:
            ev = torch.cuda.Event(enable_timing=True)
            ev.record(stream)
            record.append((None, 0, ev))

    def per_point_ms(rec):
        ms, n = [0.0] * len(gemms), [0] * len(gemms)
        for (gi, C, ev), (_, _, ev_next) in zip(rec[:-1], rec[1:]):
            ms[gi] += ev.elapsed_time(ev_next)
            n[gi] += C
        return ms, n

    def max_over_ranks(v):
        if dist is None:
            return v
        t = torch.tensor([v], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    eager_coll = world > 1 and not coll_in_graph
    run_steps(W, graphs_full, graphs_rem, eager_coll)     # W untimed warm-up steps
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
        run_steps(K_steps, graphs_full, graphs_rem, eager_coll, rec)
        t_end.record(stream)
        torch.cuda.synchronize()
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    elapsed_ms = max_over_ranks(t_start.elapsed_time(t_end))
    step_ms, step_n = per_point_ms(rec)

    # GEMM-only per-point times (N > 1: a second, shorter timed phase without the collectives)
    gemm_ms, gemm_n = step_ms, step_n
    gemm_only_ms_per_step = elapsed_ms / K_steps
    if world > 1:
        g_full = build_graphs(BLOCK_C, False)
        g_rem = build_graphs(rem, False) if rem else []
        run_steps(min(W, BLOCK_C), g_full, g_rem, False)
        torch.cuda.synchronize()
        dist.barrier()
        rec2 = []
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        run_steps(K_steps, g_full, g_rem, False, rec2)
        b.record(stream)
        torch.cuda.synchronize()
        gemm_only_ms_per_step = max_over_ranks(a.elapsed_time(b)) / K_steps
        gemm_ms, gemm_n = per_point_ms(rec2)

    peaks = load_peaks()
    ridge = peaks["tflops"] * 1e12 / (peaks["hbm_gbs"] * 1e9)
    traffic = load_traffic()
    step_flops = sum(algo_flops(g["M"], g["N"], g["K"]) for g in gemms)
    sweep = []
    for gi, g in enumerate(gemms):
        us = 1e3 * gemm_ms[gi] / max(1, gemm_n[gi])
        fl = algo_flops(g["M"], g["Nl"], g["Kl"])
        by = algo_bytes(g["M"], g["Nl"], g["Kl"], G, g["n_out"])
        tfl = fl / (us * 1e-6) / 1e12
        gbs = by / (us * 1e-6) / 1e9
        e = {"M": g["M"], "N": g["Nl"], "K": g["Kl"], "tp": g["kind"] if world > 1 else "none",
             "us": round(us, 3), "tflops": round(tfl, 2), "gbs": round(gbs, 1),
             "frac_hbm": round(gbs / peaks["hbm_gbs"], 4), "frac_tensor": round(tfl / peaks["tflops"], 4),
             "bound": "tensor" if fl / by >= ridge else "hbm", "kernel": plan_key(g["plan"]),
             "ctas": g["plan"]["num_ctas"]}
        if world > 1:
            e["us_with_collective"] = round(1e3 * step_ms[gi] / max(1, step_n[gi]), 3)
        sweep.append(e)
    layer_stack = None
    if args.workload == "mistral7b_stack":
        # per batch size: the 4 GEMMs of one layer back to back, x 32 layers
        layer_stack = []
        for M in Ms:
            key = "us_with_collective" if world > 1 else "us"
            us_layer = sum(e[key] for e in sweep if e["M"] == M)
            layer_stack.append({"M": M, "us_per_layer": round(us_layer, 3),
                                "tokens_per_s": round(M / (32 * us_layer * 1e-6), 1)})

    # roofline of the kernel that dominates the step: launches grouped by kernel identity (template
    # instantiation + schedule); the group with the largest share of the GEMM time; achieved =
    # the group's algorithmic bytes (or flops) / its measured time (a launch-weighted average)
    groups = {}
    for gi, g in enumerate(gemms):
        k = sweep[gi]["kernel"]
        d = groups.setdefault(k, {"ms": 0.0, "n": 0, "bytes": 0, "flops": 0, "t_tensor": 0.0, "points": []})
        d["ms"] += gemm_ms[gi]
        d["n"] += gemm_n[gi]
        d["bytes"] += algo_bytes(g["M"], g["Nl"], g["Kl"], G, g["n_out"]) * gemm_n[gi]
        d["flops"] += algo_flops(g["M"], g["Nl"], g["Kl"]) * gemm_n[gi]
        d["t_tensor"] += gemm_ms[gi] if sweep[gi]["bound"] == "tensor" else 0.0
        d["points"].append(f"{g['M']}x{g['Nl']}x{g['Kl']}")
    total_ms = sum(d["ms"] for d in groups.values())
    dom_key = max(groups, key=lambda k: groups[k]["ms"])
    d = groups[dom_key]
    t_s = d["ms"] * 1e-3
    clk = sampler.summary()
    # the guide's rule: the burst peak for a kernel timed alone, the sustained (power-capped) peak
    # for a kernel timed inside a long step -- a timed region of >= 0.5 s of back-to-back GEMMs, or
    # one the clock sampler saw under sw_power_cap
    sustained = elapsed_ms >= 500.0 or "sw_power_cap" in clk["reasons"]
    if d["t_tensor"] >= 0.5 * d["ms"]:
        ach = d["flops"] / t_s / 1e12
        pk = peaks["tflops_sustained"] if sustained else peaks["tflops"]
        roof = {"bound": "tensor", "achieved": round(ach, 2), "peak": pk, "unit": "TFLOP/s",
                "frac": round(ach / pk, 4), "frac_of_burst_peak": round(ach / peaks["tflops"], 4)}
    else:
        ach = d["bytes"] / t_s / 1e9
        roof = {"bound": "hbm", "achieved": round(ach, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(ach / peaks["hbm_gbs"], 4)}
    roof["traffic"] = traffic.get(f"{args.workload}:{dom_key}")
    roof["kernel"] = f"quick_w4a16_tc_kernel {dom_key}"
    roof["launches"] = d["points"]
    roof["algorithmic_per_launch"] = round((d["flops"] if roof["bound"] == "tensor" else d["bytes"]) / max(1, d["n"]))
    roof["avg_launch_us"] = round(1e3 * d["ms"] / max(1, d["n"]), 3)
    roof["peak_source"] = peaks["source"] + (", sustained figure (long timed region / power cap)" if sustained and
                                             roof["bound"] == "tensor" else ", burst figure")
    roof["share_of_step"] = round(d["ms"] / total_ms, 4)
    roof["kernel_shares"] = {k: round(v["ms"] / total_ms, 4) for k, v in sorted(groups.items(), key=lambda kv: -kv[1]["ms"])}

    # ---- e2e: through the C-ABI with host buffers (pinned), copies inside the timed region
    e2e = run_e2e(args, gemms, wcopies, R, G, stream, dist, world, quick, collective, ws)

    value = K_steps * step_flops / (elapsed_ms * 1e-3) / 1e12
    step_bytes = sum(algo_bytes(g["M"], g["Nl"], g["Kl"], G, g["n_out"]) for g in gemms) * world
    res = {
        "metric": METRIC, "value": round(value, 3), "unit": "TFLOP/s", "n_gpus": world, "steps": K_steps,
        "warmup": W, "ms_per_step": round(elapsed_ms / K_steps, 5), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic (SplitMix64 AWQ int4 weights, U[-1,1] fp16 X)",
        "config": {"workload": args.workload, "baseline_config": cfg_idx,
                   "shapes_NxK": [[n, k, kind] for n, k, kind in shapes], "M": Ms, "group_size": G,
                   "gemms_per_step": len(gemms),
                   "parallelism": (f"tp{world}: " + ", ".join(f"{n}x{k} {tp_desc(kind, peer)}" for n, k, kind in shapes))
                                   if world > 1 else "single GPU",
                   "l2": (f"rotating {R} weight copies per shape ({R * blob_bytes / 2**20:.0f} MiB) > L2 "
                          f"{l2 / 2**20:.0f} MiB; every launch reads its weights from HBM") if l2_cold else
                         f"weights L2-resident ({R} copies of {blob_bytes} B < 2.5 x L2)",
                   "timing": f"CUDA-graph replays of {BLOCK_C} launches per GEMM point (PDL between consecutive "
                             "launches), point-major; events between replays"
                             + ("; collective-fused peer-memory TP calls captured in the graphs" if peer else
                                "; NCCL collectives captured in the graphs" if coll_in_graph else
                                "; NCCL collectives eager after each replay" if world > 1 else ""),
                   "launch": "quick_w4a16_gemm_ex with QUICK_FLAG_PDL and a caller-owned stream-K workspace, "
                             "automatic plan"},
        "hbm_gbs_aggregate": round(K_steps * step_bytes / (elapsed_ms * 1e-3) / 1e9, 1),
        "gpu_launches": K_steps * sum((2 if g["kind"] == "col" else 4) if (peer and g["kind"] in ("col", "row")) else
                                      1 + (2 if (world > 1 and g["kind"] in ("col", "row")) else 0) for g in gemms),
        "roofline": roof,
        "sweep": sweep,
        **({"layer_stack_32_layers": layer_stack} if layer_stack else {}),
        **({"gemm_only_ms_per_step": round(gemm_only_ms_per_step, 5),
            "collective_ms_per_step": round(elapsed_ms / K_steps - gemm_only_ms_per_step, 5),
            "comm_nranks_ok": True} if world > 1 else {}),
        "e2e": e2e,
        "pack": {"host_seconds": round(pack_s, 4), "bytes": int(sum(l_["blob"].size for l_ in layers))},
        "clocks": clk,
    }
    return res


def run_e2e(args, gemms, wcopies, R, G, stream, dist, world, quick, collective, ws):
    import torch
    steps = max(3, min(args.steps, 100))
    out_of = [g.get("yfull", g["y"]) for g in gemms]
    xh = [torch.from_numpy(g["x_host"].view(np.int16)).view(torch.float16).pin_memory() for g in gemms]
    yh = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in out_of]
    xd = [g["xs"][0] for g in gemms]
    sh = stream.cuda_stream

    def gemm_call(gi, g, slot, x=None, y=None, w=None, s=None):
        fl = (quick.QUICK_FLAG_OUT_F32 if g["y"].dtype == torch.float32 else 0) | \
            (quick.QUICK_FLAG_SILU_MUL if g["kind"] == "silu" else 0)
        x = xd[gi] if x is None else x
        y = g["y"] if y is None else y
        w = ws if w is None else w
        quick.quick_w4a16_gemm_raw(x.data_ptr(), wcopies[g["si"]][slot].data_ptr(), g["M"], g["Nl"], g["Kl"],
                                   G, y.data_ptr(), sh if s is None else s, flags=fl, ws_ptr=w.data_ptr(),
                                   ws_bytes=w.numel(), ldy=g["n_out"])

    pipelined = world == 1
    graphs, replay_streams = [], []
    if not pipelined:
        def step(i):
            for gi, g in enumerate(gemms):
                slot = (i * len(gemms) + gi) % R
                xd[gi].copy_(xh[gi], non_blocking=True)
                gemm_call(gi, g, slot)
                collective(g)
                yh[gi].copy_(out_of[gi], non_blocking=True)
        for i in range(3):
            step(i)
        torch.cuda.synchronize()
    else:
        # Copies overlap the GEMMs, as a serving loop would run them: each step is one CUDA-graph replay
        # holding the X uploads (one copy stream), the captured C-ABI GEMM calls and the Y read-backs
        # (another copy stream) with per-GEMM event edges.  Two such graphs over two independent sets of
        # device buffers, workspaces and host read-back buffers are replayed alternately on two streams,
        # so step i + 1's uploads run while step i's last GEMMs and read-backs finish (PCIe is the bound
        # of this workload: 148 MB each way per step); a graph waits only for its own previous replay.
        s_h2d, s_d2h = torch.cuda.Stream(stream.device), torch.cuda.Stream(stream.device)
        for si in range(2):
            if si == 0:
                xs_, ys_, ws_, yh_ = xd, [g["y"] for g in gemms], ws, yh
            else:
                xs_ = [torch.empty_like(x) for x in xd]
                ys_ = [torch.empty_like(g["y"]) for g in gemms]
                ws_ = torch.zeros_like(ws)   # a concurrent replay must not share the stream-K counters
                yh_ = [torch.empty(o.shape, dtype=o.dtype).pin_memory() for o in out_of]
            rs = torch.cuda.Stream(stream.device)
            ev = {k: [torch.cuda.Event() for _ in gemms] for k in ("h2d", "comp")}
            for gi, g in enumerate(gemms):   # eager warm-up of this set's calls
                gemm_call(gi, g, gi % R, xs_[gi], ys_[gi], ws_, rs.cuda_stream)
            torch.cuda.synchronize()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph, stream=rs):
                fork = torch.cuda.Event()
                fork.record(rs)
                s_h2d.wait_event(fork)
                s_d2h.wait_event(fork)
                for gi, g in enumerate(gemms):
                    with torch.cuda.stream(s_h2d):
                        xs_[gi].copy_(xh[gi], non_blocking=True)
                        ev["h2d"][gi].record(s_h2d)
                    rs.wait_event(ev["h2d"][gi])
                    gemm_call(gi, g, (si * len(gemms) + gi) % R, xs_[gi], ys_[gi], ws_, rs.cuda_stream)
                    ev["comp"][gi].record(rs)
                    with torch.cuda.stream(s_d2h):
                        s_d2h.wait_event(ev["comp"][gi])
                        yh_[gi].copy_(ys_[gi], non_blocking=True)
                join_h, join_d = torch.cuda.Event(), torch.cuda.Event()
                join_h.record(s_h2d)
                join_d.record(s_d2h)
                rs.wait_event(join_h)
                rs.wait_event(join_d)
            graph.replay()
            torch.cuda.synchronize()
            graphs.append(graph)
            replay_streams.append(rs)
    if dist is not None:
        dist.barrier()
    def replay_steps(n, sets):
        # n steps; `sets` graphs alternate (1: every step on graph 0's stream, serialised)
        for rs in replay_streams[:sets]:
            rs.wait_event(a)
        for i in range(n):
            with torch.cuda.stream(replay_streams[i % sets]):
                graphs[i % sets].replay()
        for rs in replay_streams[:sets]:
            done = torch.cuda.Event()
            done.record(rs)
            stream.wait_event(done)

    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    sets, trial = 1, {}
    if graphs:
        # warm-up trial of both modes: the two-graph overlap wins when PCIe bounds the step (70B: 4.1 ->
        # 3.4 ms) but loses when the step is many small GEMMs that the two graphs then run concurrently
        # (4096^2: 86 -> 53 TFLOP/s); the faster one is timed
        for m in (1, 2):
            a.record(stream)
            replay_steps(4, m)
            b.record(stream)
            torch.cuda.synchronize()
            trial[m] = a.elapsed_time(b)
        sets = min(trial, key=trial.get)
    a.record(stream)
    if graphs:
        replay_steps(steps, sets)
    else:
        for i in range(steps):
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
            "h2d_bytes_per_step": int(sum(x.numel() * 2 for x in xh)),
            "d2h_bytes_per_step": int(sum(y.numel() * y.element_size() for y in yh)),
            "steps": steps, "ms_per_step": round(ms / steps, 4),
            **({"trial_ms_per_step": {("one graph" if m == 1 else "two graphs"): round(t / 4, 4) for m, t in trial.items()}}
               if graphs else {}),
            "path": ("C-ABI quick_w4a16_gemm_ex per GEMM (caller-owned workspace), pinned H2D X + D2H Y each step"
                     + ("; one CUDA-graph replay per step holding the uploads, the captured C-ABI GEMM calls and "
                        "the read-backs on three streams with event dependencies (copies overlap GEMMs)"
                        + ("; two such graphs over independent buffer sets replayed alternately on two streams "
                           "(step i+1's uploads overlap step i's tail)" if sets == 2 else
                           "; consecutive replays of one graph (faster than two alternating graphs here)")
                        if world == 1 else "; eager, with the TP collectives and epilogue kernels"))}


# ------------------------------------------------------------------------------------------ CPU arm
def oracle_step_sample(workload, budget_s):
    """Time the oracle (as it stands) on a bounded sample of one step of the workload:
    every GEMM of the step restricted to the first n_s output columns (n_s % 8 == 0)."""
    import oracle  # bench.py's cpu_baseline / reference leg is allowed to call the oracle
    _, shapes, Ms, G = WORKLOADS[workload]
    probs = []
    for si, (N, K, _kind) in enumerate(shapes):
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
                       "shapes_NxK": [[n, k, kind] for n, k, kind in shapes], "columns_per_gemm": ns},
            "cpu_baseline": {"value": round(v, 6), "unit": "TFLOP/s", "kind": "oracle", "cores": cpu_threads(),
                             "sample": sample},
            "e2e": {"value": round(v, 6), "unit": "TFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


# ------------------------------------------------------------------------------------------ main
def free_port():
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=800)
    ap.add_argument("--warmup", type=int, default=16)
    ap.add_argument("--impl", choices=["quick", "reference"], default="quick")
    ap.add_argument("--workload", choices=sorted(WORKLOADS), default=DEFAULT_WORKLOAD)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--dist-backend", choices=["nccl", "gloo"], default="nccl",
                    help="N > 1 process group: nccl (the measurement); gloo only to exercise the N > 1 code paths "
                         "with several ranks on one GPU (CUDA tensors through gloo, collectives not captured)")
    ap.add_argument("--comm", choices=["nccl", "peer"], default="nccl",
                    help="N > 1: NCCL collectives after the GEMMs, or the collective-fused peer-memory TP GEMMs")
    args = ap.parse_args()
    if args.warmup < 3 or args.steps < 1 or args.gpus < 1:
        sys.exit("bench.py: needs --warmup >= 3, --steps >= 1, --gpus >= 1")

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-launch under torchrun on this node (127.0.0.1 rendezvous)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        os.execv(sys.executable, cmd)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")

    if args.impl == "reference":
        # the oracle on the host cores: rank 0 alone runs it; the other ranks exit without work
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return

    dist = None
    if world > 1:
        import torch
        import torch.distributed as tdist
        torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)) % torch.cuda.device_count())
        tdist.init_process_group(args.dist_backend)
        if tdist.get_world_size() != args.gpus:
            sys.exit("bench.py: process group size != --gpus")
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
