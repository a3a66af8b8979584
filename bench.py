"""Benchmark of the B200 TW sparse matmul (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config bert|bert_tew|cfg1]
                    [--impl ours|reference]

One *step* = one pass of the hot path over one batch: the TW product of the
three BERT-base linear layers (768x768, 768x3072, 3072x768) at 75% TW
sparsity, G=128, M = 128 x 64 = 8192 tokens, fp16 operands, fp32
accumulation, fp16 output (configs[1]).  ``--config bert_tew`` is configs[2]
(TW 0.75 + 1.5% element overlay); ``--config cfg1`` is configs[0].

value        effective TFLOP/s = surviving FLOPs (metrics.report.sparse_flops,
             metrics.py:114-117) of all ranks / max-over-ranks device time,
             inputs resident in HBM; 4 rotating buffer sets (> 2 x L2) so
             every step streams cold activations, weights and outputs.  The
             timed steps replay one CUDA graph per rotation (4 steps = 12
             layer launches chained by programmatic dependent launch); the
             dense cuBLAS arm is graph-captured the same way.
             Activations are resident as A^T (K x M, tokens contiguous): the
             layout K1 reads and writes (a TW layer's C'^T output is the next
             layer's A^T); the cuBLAS arm reads the same A^T buffers.
transpose    A (M x K row-major, device) -> A^T (K4, tw_transpose_cast) per
             step, reported beside value for callers holding row-major
             activations (value_incl_transpose).
e2e          same metric through the public API (TwPlan.prepare + TwPlan.run)
             from pinned HOST fp16 activations (M x K, the reference's layout),
             with the H2D copies, the A -> A^T kernel (K4), the GEMM and the
             D2H copy of the fp16 result inside the timed region.
cublas       dense torch.matmul (cuBLAS) at the same shapes and layout.
roofline     K1 (tw_gemm_kernel) launches timed per layer with CUDA events;
             achieved = algorithmic bytes / launch time vs the
             measured HBM peak (the step is HBM-bound: AI 188 < ridge 240).
cpu_baseline the reference algorithm (oracle port of execute_batched,
             executor.py:230-265) on host cores, bounded M-slice sample.

N > 1 (torchrun): weak scaling, every rank runs its own 8192-token batch
(M-split data parallelism, no collective on the data path).
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "TW-GEMM speedup vs dense cuBLAS at 75% sparsity; effective TFLOP/s"
BERT_LAYERS = [(768, 768), (768, 3072), (3072, 768)]
CONFIGS = {
    "bert": {"layers": BERT_LAYERS, "m": 8192, "s": 0.75, "g": 128, "delta": 0.0,
             "workload": "BERT-base linear layers 768x768, 768x3072, 3072x768; TW 75% G=128; "
                         "M=128x64 tokens; fp16 (configs[1])"},
    "bert_tew": {"layers": BERT_LAYERS, "m": 8192, "s": 0.75, "g": 128, "delta": 0.015,
                 "workload": "BERT-base TEW: TW 75% + 1.5% element overlay, G=128, "
                             "M=8192 (configs[2])"},
    "bert_tvw": {"layers": BERT_LAYERS, "m": 8192, "s": 0.75, "g": 128, "delta": 0.0,
                 "pattern": "tvw",
                 "workload": "BERT-base TVW: TW at 50% then 2:4 down every payload column "
                             "(75% total), G=128, M=8192 (SURVEY 8f1; dense UMMA over the "
                             "2:4 payload)"},
    "cfg1": {"layers": [(1024, 1024)], "m": 128, "s": 0.75, "g": 128, "delta": 0.0,
             "workload": "single 1024x1024 weight, TW 75% G=128, M=128 (configs[0])"},
    "big": {"layers": [(16384, 16384)], "m": 8192, "s": 0.75, "g": 128, "delta": 0.0,
            "workload": "16384x16384 TW 75% G=128, M=8192; column tiles sharded over the "
                        "ranks + NCCL all-gather of C'^T (configs[4])"},
}
N_ROTATE = 4


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm": float(d["hbm_gbs"]), "tc": float(d["bf16_tflops"]),
                "tc_sustained": float(d.get("bf16_tflops_sustained", d["bf16_tflops"])),
                "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm": 6650.0, "tc": 1590.0, "tc_sustained": 1400.0,
            "source": "fallback (B200_PROFILING.md)"}


# ----------------------------------------------------------------------------
# clocks sampler
# ----------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 8:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[4:8]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx),
                "reasons": sorted(reasons), "samples": len(sm)}


# ----------------------------------------------------------------------------
# problem construction (host prune/compress, identical on every rank)
# ----------------------------------------------------------------------------

def build_layers(cfg: dict):
    import paper_2402_10876_b200 as tw

    layers = []
    for li, (k, n) in enumerate(cfg["layers"]):
        w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
        if cfg["delta"] > 0:
            plan, tsm, ov = tw.prune_tew(w, cfg["s"], cfg["delta"], cfg["g"])
        elif cfg.get("pattern") == "tvw":
            plan, tsm, _ = tw.prune_tvw(w, cfg["s"], cfg["g"])
            ov = None
        else:
            plan, tsm = tw.prune_tw(w, cfg["s"], cfg["g"])
            ov = None
        enc = tw.encode_cto(tsm)
        n_out = tsm.n_condensed
        if ov is not None:
            ov_cols = np.flatnonzero(np.diff(ov.col_ptr))
            n_out = int(np.union1d(tsm.column_mask.kept, ov_cols).size)
        layers.append({"k": k, "n": n, "w": w, "plan": plan, "tsm": tsm, "enc": enc, "ov": ov,
                       "flops": tw.sparse_flops(tsm, cfg["m"], ov),
                       "bytes": tw.algorithmic_bytes(tsm, cfg["m"], overlay=ov, n_out=n_out)})
    return layers


def activations(cfg: dict, k: int, li: int, rank: int):
    import paper_2402_10876_b200 as tw

    # stream 1 = input stream of the reference CLI; each rank its own batch
    return tw.round_to(tw.synthetic_matrix(rank, cfg["m"], k, tw.STREAM_INPUT), "fp16")


# ----------------------------------------------------------------------------
# reference arm / CPU baseline: the reference algorithm on host cores
# ----------------------------------------------------------------------------

def cpu_model() -> str:
    """Host CPU model name (for the cpu_baseline record)."""
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_reference_rate(cfg: dict, layers, m_sample: int, reps: int = 1, workers: int = 0):
    """Time the oracle port of execute_batched (+ gemm_tew overlay) on an
    M-slice with `workers` lanes (0: every host core); returns (TFLOP/s,
    seconds, flops, workers)."""
    from oracle import tilesparse_oracle as orc

    workers = workers or os.cpu_count() or 1
    total_s, total_f = 0.0, 0
    for _ in range(reps):
        for li, L in enumerate(layers):
            a = activations(cfg, L["k"], li, 0)[:m_sample]
            tiles = [(t.kept_rows.kept, t.payload) for t in L["tsm"].tiles]
            t0 = time.perf_counter()
            out = orc.execute_batched(a, tiles, workers, "lpt")
            if L["ov"] is not None and L["ov"].nnz:
                full = np.zeros((a.shape[0], L["n"]))
                full[:, L["tsm"].column_mask.kept] = out
                orc.gemm_tew_add(a, full, L["ov"].col_ptr, L["ov"].row_idx, L["ov"].values)
            total_s += time.perf_counter() - t0
            nnz = L["ov"].nnz if L["ov"] is not None else 0
            total_f += 2 * m_sample * (sum(t.width * t.kept_rows.n_kept for t in L["tsm"].tiles)
                                       + nnz)
    return total_f / total_s / 1e12, total_s, total_f, workers


def run_reference_arm(args, cfg, rank: int, world: int) -> None:
    if rank != 0:
        return
    layers = build_layers(cfg)
    m_sample = min(cfg["m"], 512)
    for _ in range(args.warmup):
        cpu_reference_rate(cfg, layers, m_sample)
    rate, secs, flops, workers = cpu_reference_rate(cfg, layers, m_sample, reps=args.steps)
    sample = (f"{m_sample} of {cfg['m']} tokens per step through every layer "
              f"(oracle port of execute_batched, lpt, {workers} workers)")
    line = {
        "metric": METRIC, "value": rate, "unit": "TFLOP/s", "impl": "reference",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": secs / args.steps * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (Philox seed 0, fp16-rounded)",
        "config": {"workload": cfg["workload"], "parallelism": "cpu", "m_sample": m_sample},
        "cpu_baseline": {"cpu_model": cpu_model(), "value": rate, "unit": "TFLOP/s", "cores": workers, "kind": "port",
                         "sample": sample},
        "e2e": {"value": rate, "unit": "TFLOP/s", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------
# our arm
# ----------------------------------------------------------------------------

def ncu_traffic(config: str):
    """DRAM bytes per step of the product kernels, from the committed ncu
    launch lists (profiles/ncu_traffic.json, scripts/ncu_traffic.sh); None
    when not captured for this config."""
    tfile = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(tfile.read_text()).get(config)
    except (ValueError, OSError):
        return None


def capture_graph(fn):
    """CUDA graph of fn() (eager warm-up first, captured on a side stream)."""
    import torch

    g = torch.cuda.CUDAGraph()
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(side):
        fn()
        with torch.cuda.graph(g, stream=side):
            fn()
    torch.cuda.current_stream().wait_stream(side)
    torch.cuda.synchronize()
    return g


def run_ours(args, cfg, rank: int, world: int) -> None:
    import torch
    import torch.distributed as dist

    import paper_2402_10876_b200 as tw

    dev = torch.device("cuda", torch.cuda.current_device())
    layers = build_layers(cfg)
    m = cfg["m"]
    tew = cfg["delta"] > 0

    # R rotating sets of (plan, A^T, C^T) per layer: total footprint > 2 x L2
    sets = []
    for r in range(N_ROTATE):
        layer_set = []
        for li, L in enumerate(layers):
            # activations in the plan's row-run layout (prepare() writes it;
            # TEW plans read it in K1 and K2)
            plan = tw.TwPlan(L["enc"], L["ov"], compute_dtype="fp16", row_layout="runs")
            a = activations(cfg, L["k"], li, rank)
            at = plan.prepare(torch.from_numpy(a).to(dev))
            rows = plan.info.n_union if tew else plan.info.n_condensed
            ct = torch.empty((rows, m), dtype=torch.float16, device=dev)
            layer_set.append((plan, at, ct))
        sets.append(layer_set)
    torch.cuda.synchronize()

    def run_set(r: int):
        for plan, at, ct in sets[r]:
            if tew:
                plan.run_tew(at, out=ct)
            else:
                plan.run(at, out=ct)

    # one CUDA graph per rotating set: a step is one graph replay (3 launches)
    graphs = [capture_graph(lambda r=r: run_set(r)) for r in range(N_ROTATE)]
    # one graph of a whole rotation (N_ROTATE steps): programmatic dependent
    # launch chains every kernel of it, not only the three inside a step
    cycle = capture_graph(lambda: [run_set(r) for r in range(N_ROTATE)])

    def step(i: int):
        graphs[i % N_ROTATE].replay()

    def run_steps(n: int):
        """n steps starting at set 0: whole rotations as one replay each."""
        for _ in range(n // N_ROTATE):
            cycle.replay()
        for i in range(n % N_ROTATE):
            step(i)

    flops_step = sum(L["flops"] for L in layers)
    stream = torch.cuda.current_stream()

    # ---- timed region: K steps, barrier + sync on both sides, max over ranks
    with ClockSampler(torch.cuda.current_device()) as clk:
        # soak so the clock sampler sees the GPU under this load (>= ~1 s)
        t_soak = time.time()
        i = 0
        while time.time() - t_soak < 1.0:
            step(i)
            i += 1
            if i % 64 == 0:
                torch.cuda.synchronize()
        for i in range(args.warmup):
            step(i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        run_steps(args.steps)
        ev1.record(stream)
        torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    ms = ev0.elapsed_time(ev1)
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_max = float(t.item())
    ms_step = ms_max / args.steps
    value = world * flops_step / (ms_step * 1e-3) / 1e12

    # ---- per-launch K1 timing (roofline): graph of REPS launches per layer
    per_layer = []
    reps = 32
    for li, L in enumerate(layers):
        def layer_launches(li=li):
            for i in range(reps):
                plan, at, ct = sets[i % N_ROTATE][li]
                if tew:
                    plan.run_tew(at, out=ct)
                else:
                    plan.run(at, out=ct)
        g = capture_graph(layer_launches)
        times = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            g.replay()
            e1.record(stream)
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e3 / reps)
        us = statistics.median(times)
        per_layer.append({"shape": f"{L['k']}x{L['n']}", "us": us, "flops": L["flops"],
                          "bytes": L["bytes"],
                          "tflops": L["flops"] / (us * 1e-6) / 1e12,
                          "gbs": L["bytes"] / (us * 1e-6) / 1e9})
        del g

    # ---- dense cuBLAS at the same shapes / layout (C^T = W^T . A^T)
    dense = []
    for r in range(N_ROTATE):
        row = []
        for li, L in enumerate(layers):
            wt = torch.from_numpy(np.ascontiguousarray(L["w"].T)).to(dev, torch.float16)
            a_nat = activations(cfg, L["k"], li, rank)
            at_nat = tw.prepare_activations(torch.from_numpy(a_nat).to(dev))  # plain A^T
            row.append((wt, at_nat,
                        torch.empty((L["n"], m), dtype=torch.float16, device=dev)))
        dense.append(row)

    def dense_set(r: int):
        for wt, at, out in dense[r]:
            torch.matmul(wt, at, out=out)

    dense_graphs = [capture_graph(lambda r=r: dense_set(r)) for r in range(N_ROTATE)]
    dense_cycle = capture_graph(lambda: [dense_set(r) for r in range(N_ROTATE)])

    def dense_step(i: int):
        dense_graphs[i % N_ROTATE].replay()

    for i in range(args.warmup):
        dense_step(i)
    torch.cuda.synchronize()
    d0, d1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    d0.record(stream)
    for _ in range(args.steps // N_ROTATE):   # same graph structure as our arm
        dense_cycle.replay()
    for i in range(args.steps % N_ROTATE):
        dense_step(i)
    d1.record(stream)
    torch.cuda.synchronize()
    dense_ms = d0.elapsed_time(d1) / args.steps
    td = torch.tensor([dense_ms], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(td, op=dist.ReduceOp.MAX)
    dense_ms = float(td.item())
    dense_flops = sum(2 * m * L["k"] * L["n"] for L in layers)
    del dense, dense_graphs

    # ---- row-major callers: A (M x K, fp16, device) -> A^T per layer (K4)
    a_dev = [torch.from_numpy(activations(cfg, L["k"], li, rank)).to(dev, torch.float16)
             for li, L in enumerate(layers)]

    def prep_set(r: int):
        for li, (plan, at, _) in enumerate(sets[r]):
            plan.prepare(a_dev[li], out=at)

    prep_graphs = [capture_graph(lambda r=r: prep_set(r)) for r in range(N_ROTATE)]
    p0, p1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    p0.record(stream)
    for i in range(args.steps):
        prep_graphs[i % N_ROTATE].replay()
    p1.record(stream)
    torch.cuda.synchronize()
    prep_ms = p0.elapsed_time(p1) / args.steps
    del prep_graphs

    # ---- e2e through the public API from pinned host memory: per layer
    # H2D of A (M x K fp16, the reference layout) -> prepare (K4) -> run (K1
    # [+ K2]) -> D2H of the native C'^T.  Three streams pipeline the layers:
    # the copy engines (H2D, D2H: full duplex) overlap each other and the
    # kernels; events order every reuse of a device buffer.
    host_a = [torch.from_numpy(activations(cfg, L["k"], li, rank)).to(torch.float16)
              .pin_memory() for li, L in enumerate(layers)]
    host_c = [torch.empty(tuple(s[2].shape), dtype=torch.float16).pin_memory()
              for s in sets[0]]
    dev_a = [[torch.empty(h.shape, dtype=torch.float16, device=dev) for h in host_a]
             for _ in range(2)]
    h2d = sum(h.numel() * h.element_size() for h in host_a)
    d2h = sum(h.numel() * h.element_size() for h in host_c)
    s_in, s_out = torch.cuda.Stream(), torch.cuda.Stream()
    nl = len(layers)
    ev = lambda: torch.cuda.Event()  # noqa: E731
    ev_in = [[ev() for _ in range(nl)] for _ in range(2)]
    ev_comp = [[ev() for _ in range(nl)] for _ in range(2)]
    ev_out = [[ev() for _ in range(nl)] for _ in range(N_ROTATE)]
    for e_list in ev_comp + ev_out:
        for e_ in e_list:
            e_.record(stream)

    def e2e_step(i: int):
        p, r = i % 2, i % N_ROTATE
        for li in range(nl):
            s_in.wait_event(ev_comp[p][li])        # dev_a[p][li] consumed two steps ago
            with torch.cuda.stream(s_in):
                dev_a[p][li].copy_(host_a[li], non_blocking=True)
                ev_in[p][li].record(s_in)
        for li, (plan, _, ct) in enumerate(sets[r]):
            stream.wait_event(ev_in[p][li])
            stream.wait_event(ev_out[r][li])       # ct's previous D2H is done
            at = plan.prepare(dev_a[p][li])
            if tew:
                plan.run_tew(at, out=ct)
            else:
                plan.run(at, out=ct)
            ev_comp[p][li].record(stream)
            s_out.wait_event(ev_comp[p][li])
            with torch.cuda.stream(s_out):
                host_c[li].copy_(ct, non_blocking=True)
                ev_out[r][li].record(s_out)

    for i in range(args.warmup):
        e2e_step(i)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    s_in.wait_event(e0)
    s_out.wait_event(e0)
    for i in range(args.steps):
        e2e_step(i)
    stream.wait_stream(s_out)
    e1.record(stream)
    torch.cuda.synchronize()
    te = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=dev)
    if world > 1:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    e2e_ms = float(te.item()) / args.steps
    e2e_value = world * flops_step / (e2e_ms * 1e-3) / 1e12

    if rank != 0:
        return

    pk = peaks()
    tot_bytes = sum(p["bytes"] for p in per_layer)
    tot_us = sum(p["us"] for p in per_layer)
    achieved_gbs = tot_bytes / (tot_us * 1e-6) / 1e9
    ai = flops_step / tot_bytes
    ridge = pk["tc"] * 1e12 / (pk["hbm"] * 1e9)
    traffic = ncu_traffic(args.config)
    if ai < ridge:
        roofline = {"bound": "hbm", "achieved": achieved_gbs, "peak": pk["hbm"], "unit": "GB/s",
                    "frac": achieved_gbs / pk["hbm"], "traffic": traffic}
    else:
        tf = flops_step / (tot_us * 1e-6) / 1e12
        roofline = {"bound": "tensor", "achieved": tf, "peak": pk["tc"], "unit": "TFLOP/s",
                    "frac": tf / pk["tc"], "traffic": traffic}
    roofline.update({"kernel": "tw_gemm_kernel" + ("+tw_residual_kernel" if tew else ""),
                     "peak_source": pk["source"], "arithmetic_intensity": ai,
                     "layers": per_layer})

    # CPU baseline: the reference algorithm on this host, bounded sample
    m_sample = min(m, 1024)
    cpu_rate, cpu_s, _, workers = cpu_reference_rate(cfg, layers, m_sample)
    # the single-lane figure (W = 1, as cmd_bench's default) on a quarter sample
    cpu1_rate, cpu1_s, _, _ = cpu_reference_rate(cfg, layers, max(64, m_sample // 4), workers=1)
    clocks = clk.summary()
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic (Philox seed=rank, fp16-rounded; weights seed 0)",
        "config": {"workload": cfg["workload"], "m_tokens_per_gpu": m,
                   "sparsity": cfg["s"], "g": cfg["g"], "delta": cfg["delta"],
                   "parallelism": f"dp{world} (M-split, no collective)",
                   "l2": f"{N_ROTATE} rotating buffer sets (weights, A^T, C^T) > 2x L2"},
        "speedup_vs_cublas": dense_ms / ms_step,
        "transpose": {"ms_per_step": prep_ms,
                 "what": "A (M x K fp16, device, row-major) -> A^T per layer (TwPlan.prepare: K4 + row order); "
                         "only for row-major callers (a TW layer's C'^T output is already the "
                         "next layer's A^T); inside e2e",
                 "value_incl_transpose": world * flops_step / ((ms_step + prep_ms) * 1e-3) / 1e12,
                 "speedup_vs_cublas_incl_transpose": dense_ms / (ms_step + prep_ms)},
        "cublas": {"ms_per_step": dense_ms,
                   "tflops_dense": world * dense_flops / (dense_ms * 1e-3) / 1e12},
        "frac_of_dense_peak": value / world / pk["tc"],
        "e2e": {"value": e2e_value, "unit": "TFLOP/s", "ms_per_step": e2e_ms,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "path": "pinned host fp16 A (M x K) -> H2D -> TwPlan.prepare (K4) -> TwPlan.run "
                        "(K1) -> D2H of the fp16 C'^T; layers pipelined over H2D / compute / "
                        "D2H streams"},
        "roofline": roofline,
        "cpu_baseline": {"cpu_model": cpu_model(), "value": cpu_rate, "unit": "TFLOP/s", "cores": workers, "kind": "port",
                         "sample": f"{m_sample} of {m} tokens through every layer "
                                   f"({cpu_s:.1f} s, oracle port of execute_batched lpt)",
                         "value_1_worker": cpu1_rate,
                         "sample_1_worker": f"{max(64, m_sample // 4)} tokens, 1 lane ({cpu1_s:.1f} s)"},
        "gpu_launches": args.steps * len(layers) * (2 if tew else 1),
        "launch": "CUDA graph per step (one graph per rotating buffer set)",
        "clocks": clocks,
    }
    print(json.dumps(line))


# ----------------------------------------------------------------------------
# configs[4]: one large layer, column tiles sharded across ranks (strong scaling)
# ----------------------------------------------------------------------------

def run_big(args, cfg, rank: int, world: int) -> None:
    """16384^2 TW layer, M=8192.  Rank r owns a contiguous, MAC-balanced group
    of column tiles (distributed.column_shards), runs K1 on it and one
    all_gather_into_tensor assembles the full C'^T (N' x M).  A step = K1 on
    the shard + the all-gather; value = the WHOLE layer's surviving FLOPs /
    max-over-ranks step time (strong scaling).  Inputs (268 MB A^T, 134 MB
    payload, 134 MB output per rank) exceed L2, so there is no rotation."""
    import torch
    import torch.distributed as dist

    import paper_2402_10876_b200 as tw
    from paper_2402_10876_b200 import distributed as D

    dev = torch.device("cuda", torch.cuda.current_device())
    (k, n), m = cfg["layers"][0], cfg["m"]
    w = tw.round_to(tw.synthetic_matrix(0, k, n, tw.STREAM_WEIGHTS), "fp16")
    _, tsm = tw.prune_tw(w, cfg["s"], cfg["g"])
    enc = tw.encode_cto(tsm)
    shards = D.column_shards(enc, world)
    rows = D.shard_rows(enc, shards)
    lo, hi = shards[rank]
    plan = tw.TwPlan(D.shard_encoding(enc, lo, hi), compute_dtype="fp16")
    flops_total = tw.sparse_flops(tsm, m)
    flops_local = plan.flops(m)
    a_host = tw.round_to(tw.synthetic_matrix(0, m, k, tw.STREAM_INPUT), "fp16")
    a_dev = torch.from_numpy(a_host).to(dev, torch.float16)
    at = plan.prepare(a_dev)
    r0, r1 = rows[rank]
    tallest = max(b - a for a, b in rows)
    local = torch.empty((tallest, m), dtype=torch.float16, device=dev)
    full = torch.empty((tallest * world, m), dtype=torch.float16, device=dev)
    stream = torch.cuda.current_stream()

    def step(i: int = 0):
        plan.run(at, out=local[: r1 - r0])
        if world > 1:
            dist.all_gather_into_tensor(full, local)

    def timed(fn, steps):
        for i in range(args.warmup):
            fn(i)
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for i in range(steps):
            fn(i)
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1) / steps], dtype=torch.float64, device=dev)
        if world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    with ClockSampler(torch.cuda.current_device()) as clk:
        t_soak = time.time()
        while time.time() - t_soak < 1.0:
            step()
            torch.cuda.synchronize()
        ms_step = timed(step, args.steps)
    value = flops_total / (ms_step * 1e-3) / 1e12

    # K1 alone on this rank's shard (roofline) and the all-gather alone
    ms_k1 = timed(lambda i: plan.run(at, out=local[: r1 - r0]), args.steps)
    ms_ag = timed(lambda i: dist.all_gather_into_tensor(full, local), args.steps) if world > 1 else 0.0

    # dense cuBLAS on the same column share (N/world columns of W, same A^T)
    c0 = n * rank // world
    c1 = n * (rank + 1) // world
    wt = torch.from_numpy(np.ascontiguousarray(w[:, c0:c1].T)).to(dev, torch.float16)
    at_plain = tw.prepare_activations(a_dev)
    dense_out = torch.empty((c1 - c0, m), dtype=torch.float16, device=dev)
    ms_dense = timed(lambda i: torch.matmul(wt, at_plain, out=dense_out), args.steps)
    del wt, dense_out

    # e2e through the public API: pinned host A (M x K) -> H2D -> K4 -> K1 ->
    # all-gather -> D2H of the full fp16 C'^T
    a_pin = torch.from_numpy(a_host).to(torch.float16).pin_memory()
    c_pin = torch.empty((tallest * world if world > 1 else r1 - r0, m),
                        dtype=torch.float16).pin_memory()

    def e2e(i: int = 0):
        a_dev.copy_(a_pin, non_blocking=True)
        x = plan.prepare(a_dev)
        plan.run(x, out=local[: r1 - r0])
        if world > 1:
            dist.all_gather_into_tensor(full, local)
            c_pin.copy_(full, non_blocking=True)
        else:
            c_pin.copy_(local[: r1 - r0], non_blocking=True)

    ms_e2e = timed(e2e, max(2, args.steps // 4))
    if rank != 0:
        return
    pk = peaks()
    tf_k1 = flops_local / (ms_k1 * 1e-3) / 1e12
    roofline = {"bound": "tensor", "achieved": tf_k1, "peak": pk["tc"], "unit": "TFLOP/s",
                "frac": tf_k1 / pk["tc"],
                "traffic": ncu_traffic(args.config) if world == 1 else None,
                "kernel": "tw_gemm_kernel",
                "peak_source": pk["source"],
                "arithmetic_intensity": flops_total / tw.algorithmic_bytes(tsm, m),
                "k1_ms": ms_k1, "allgather_ms": ms_ag}
    # CPU baseline: the reference algorithm on one tile over 64 tokens, scaled
    from oracle import tilesparse_oracle as orc
    t = tsm.tiles[0]
    a_s = a_host[:64]
    t0 = time.perf_counter()
    orc.execute_batched(a_s, [(t.kept_rows.kept, t.payload)], os.cpu_count() or 1, "lpt")
    cpu_s = time.perf_counter() - t0
    cpu_rate = 2 * 64 * t.width * t.kept_rows.n_kept / cpu_s / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": "TFLOP/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "fp16",
        "data": "synthetic (Philox seed 0, fp16-rounded)",
        "config": {"workload": cfg["workload"], "m_tokens": m, "sparsity": cfg["s"],
                   "g": cfg["g"], "parallelism": f"column tiles / {world} ranks + all-gather",
                   "l2": "inputs > L2 (268 MB A^T, 134 MB payload, 134 MB C'^T)"},
        "speedup_vs_cublas": ms_dense / ms_k1,
        "cublas": {"ms_per_step": ms_dense, "columns_per_rank": c1 - c0,
                   "tflops_dense": 2 * m * k * (c1 - c0) / (ms_dense * 1e-3) / 1e12},
        "frac_of_dense_peak": tf_k1 / pk["tc"],
        "e2e": {"value": flops_total / (ms_e2e * 1e-3) / 1e12, "unit": "TFLOP/s",
                "ms_per_step": ms_e2e, "h2d_bytes_per_step": a_pin.numel() * 2,
                "d2h_bytes_per_step": c_pin.numel() * 2,
                "path": "pinned host fp16 A -> H2D -> K4 -> K1 -> all-gather -> D2H"},
        "roofline": roofline,
        "cpu_baseline": {"cpu_model": cpu_model(), "value": cpu_rate, "unit": "TFLOP/s", "cores": os.cpu_count() or 1,
                         "kind": "port", "sample": f"tile 0 (K'={t.kept_rows.n_kept}) x 64 tokens "
                                                   f"({cpu_s:.1f} s, one lane: one tile)"},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    print(json.dumps(line))


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="bert", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))

    if args.impl == "reference":
        run_reference_arm(args, cfg, rank, world)
        return

    import torch
    import torch.distributed as dist

    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.config == "big":
            run_big(args, cfg, rank, world)
        else:
            run_ours(args, cfg, rank, world)
    finally:
        if world > 1:
            dist.destroy_process_group()


if __name__ == "__main__":
    main()
