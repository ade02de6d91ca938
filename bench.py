#!/usr/bin/env python3
"""bench.py -- hot-path benchmark of the B200-native accumulated-update H-matrix
product (BASELINE.json configs[3], "config 4"):

    Z <- blocktrunc(Z + X Y),  X = Y = Z = H-matrix of the BEM-like kernel on
    the level-6 refined icosahedron (n = 81920), leaf 64, eta 2, eps 1e-6.

One STEP = one hm_addmul (all of SURVEY §8(a) rows A1-A6: plan, addproduct
evaluation, TRUNC, split restriction, terminal flush, virtual recursion +
rkmerge) on fresh clones of the resident H-matrix.  `value` = convention
FP64 GFLOP/s of the batched low-rank update work over the
device-timed region; `e2e` = same flops with host descriptions uploaded /
the result downloaded through the C-ABI inside the timed region.

The line also carries (BASELINE.json metric, first half): H-LR / H-Cholesky
setup seconds and convention GFLOP/s at configs[1], configs[2], the metric's
n = 81920 H-LR ("config 4'") and configs[4] (n = 327680); the standalone
batched flush (captured in situ + synthetic prescribed-sigma stacks); the
roofline of the top kernel functions; the standard (S0) product next to the
accumulated one when available; the CPU oracle on all host cores.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4|1] [--no-cpu-baseline] [--no-factor] [--no-flush] [--no-s0]

`--impl reference` times the CPU oracle (oracle/, the reference arm of this
tier) on a bounded sample of the same workload; it is test infrastructure,
never on the product path.
"""
from __future__ import annotations

import os

# the CPU oracle legs fork one single-threaded worker per core: pin BLAS to one
# thread BEFORE numpy is imported anywhere (otherwise every worker runs a
# core-count OpenBLAS pool and the host is oversubscribed)
os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
os.environ.setdefault("OMP_NUM_THREADS", "1")

import argparse
import json
import socket
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

CONFIGS = {
    # BASELINE.json configs[3] (bench workload) and configs[0] (oracle-sized)
    4: dict(level=6, leaf=64, eta=2.0, eps=1e-6, name="cfg4 hm_addmul Z<-Z+XY n=81920 (icosphere L6) leaf64 eta2 eps1e-6"),
    1: dict(level=3, leaf=32, eta=2.0, eps=1e-4, name="cfg1 hm_addmul Z<-Z+XY n=1280 (icosphere L3) leaf32 eta2 eps1e-4"),
}
METRIC = "batched low-rank update FP64 GFLOP/s (hm_addmul, accumulated updates)"
# (key, icosphere level, leaf, eps, kernel 0=G 1=(G+G^T)/2, op, repetitions)
FACTOR_RUNS = [
    ("cfg2_hlr_n5120", 4, 32, 1e-4, 0, "lr", 2),
    ("cfg3_hchol_n20480", 5, 32, 1e-5, 1, "chol", 1),
    ("cfg4p_hlr_n81920", 6, 64, 1e-6, 0, "lr", 1),
    ("cfg5_hlr_n327680", 7, 64, 1e-4, 0, "lr", 1),
]
# profile class -> (kernel function, bound, what the class's convention work measures)
CLASS_FUNCTION = {
    "qr": ("k_qr_reg+k_qr_blocked+k_qr (Householder QR of the stacks, incl. TSQR)", "alu"),
    "jacobi_svd": ("k_svd (QRCP + one-sided Jacobi)", "alu"),
    "trunc_fused": ("k_trunc_small (fused TRUNC)", "alu"),
    "eval": ("k_eval2 (H x thin dense, addeval)", "hbm"),
    "apply_q": ("k_applyq_dmma+k_applyq (reform A' = Q_A U)", "alu"),
    "gemm_M": ("k_gemm2 (M = R_A R_B^T)", "alu"),
    "dense_add": ("k_gemm2 (dense flush N += A B^T)", "alu"),
    "copy": ("k_copy (stack gathers)", "hbm"),
    "pre_qr_M": ("k_qr_blocked (pre-QR of large M)", "alu"),
}
NCU_NAME = {"qr": "k_qr_reg+k_qr_blocked+k_qr", "jacobi_svd": "k_svd", "trunc_fused": "k_trunc_small",
            "eval": "k_eval2", "apply_q": "k_applyq_dmma+k_applyq", "gemm_M": "k_gemm2", "dense_add": "k_gemm2",
            "copy": "k_copy", "pre_qr_M": "k_qr_reg+k_qr_blocked"}


def ncu_function(tj, names):
    """dram bytes per launch over the kernel functions `a+b+...` of one class
    (profiles/*_traffic.json, scripts/ncu_traffic.py)."""
    launches = byts = 0.0
    for n in names.split("+"):
        f = tj.get(n)
        if f:
            launches += f["launches"]
            byts += f.get("dram_bytes", f["dram_bytes_per_launch"] * f["launches"])
    return {"dram_bytes_per_launch": byts / launches} if launches else {}
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # DFMA/DMMA: SMs x FMA/clk x 2 x max clock
CPU_SAMPLE_LEVEL = 5   # oracle sample: icosphere L5 (n = 20480) with config 4's leaf / eta / eps


T0 = time.time()


def log(msg):
    print(f"[bench {time.time() - T0:7.1f}s] {msg}", file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons DURING the timed region."""

    FIELDS = "clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown," \
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap"

    def __init__(self, index):
        self.index = index
        self.samples = []
        self.stop = threading.Event()
        self.t = None

    def _run(self):
        while not self.stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.samples.append([x.strip() for x in out.split(",")])
            except Exception:
                pass
            self.stop.wait(0.2)

    def __enter__(self):
        self.t = threading.Thread(target=self._run, daemon=True)
        self.t.start()
        return self

    def __exit__(self, *a):
        self.stop.set()
        if self.t:
            self.t.join(timeout=10)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if "Active" in s[2 + i] and "Not" not in s[2 + i]})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def max_over_ranks(ms, device=None):
    """Device time of the timed region as the MAX over ranks (replicas: the
    job ends when the slowest rank ends).  Single process: unchanged."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(ms)
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_value(world_size, flops_per_rank_step, ms_per_step):
    """`value` = the units ALL ranks processed / the (max-over-ranks) time:
    every replica runs the same product, so ws x its convention flops."""
    return world_size * flops_per_rank_step / (ms_per_step * 1e-3) / 1e9


def measure_dgemm_tflops(torch, dev):
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device=dev)
    b = torch.randn(n, n, dtype=torch.float64, device=dev)
    for _ in range(2):
        torch.matmul(a, b)
    torch.cuda.synchronize(dev)
    best = 1e30
    for _ in range(5):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    del a, b
    return 2.0 * n ** 3 / (best * 1e-3) / 1e12


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def trunc_flops(m, n, l, k):
    """SURVEY §8(d) convention flops of one truncation (same formula as libhm's
    trunc_flops and oracle/flops.py)."""
    if l <= 0:
        return 0.0
    if l < min(m, n):
        return 2.0 * (m + n) * l * l - (4.0 / 3.0) * l ** 3 + l ** 3 / 3.0 + 22.0 * l ** 3 + 2.0 * (m + n) * l * k
    p, q = max(m, n), min(m, n)
    return 2.0 * m * n * l + 14.0 * p * q * q + 8.0 * q ** 3


# ---------------------------------------------------------------- CPU leg
def oracle_sample(cfg, cores, level=CPU_SAMPLE_LEVEL, prebuilt=None):
    """The oracle (as it stands) on a bounded sample of the same workload: the
    S2 accumulated product (oracle.parallel.addmul_s2_parallel: the serial
    oracle's arithmetic, independent subtrees on a process pool, pinned
    bit-identical to oracle.product.addmul_s2 by tests/test_oracle_parallel.py)
    on the level-`level` icosphere with the config's leaf size, eta and eps, on
    `cores` host cores.  Returns (GFLOP/s, seconds, sample text, GFLOP, build)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from hm_inputs import sphere_points
    from oracle.hmatrix import Problem
    from oracle.parallel import addmul_s2_parallel, build_parallel

    L = min(cfg["level"], level)
    if prebuilt is None:
        x, w = sphere_points(L)
        P = Problem(x, w, cfg["leaf"], cfg["eta"])
        G = build_parallel(P, cfg["eps"], cores)
        prebuilt = (P, G)
    P, G = prebuilt
    t0 = time.perf_counter()
    Z, info = addmul_s2_parallel(1.0, G.clone(), G.clone(), G.clone(), cfg["eps"], workers=cores, frontier_depth=4)
    dt = time.perf_counter() - t0
    gf = info["conv_gflop"]   # SURVEY §8(d) convention work (oracle/flops.py), printed-branch widths
    sample = (f"oracle S2 product (oracle.parallel.addmul_s2_parallel, NumPy/OpenBLAS 1 thread per worker, "
              f"{cores} worker processes) on the n={P.ct.n} icosphere (L={L}) with leaf {cfg['leaf']}, "
              f"eta {cfg['eta']}, eps {cfg['eps']:g}: {gf:.1f} convention GFLOP in {dt:.1f} s")
    return gf / dt, dt, sample, gf, prebuilt


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cores = host_cores()
    times, rates = [], []
    sample = ""
    pre = None
    for i in range(args.warmup + args.steps):
        rate, dt, sample, gf, pre = oracle_sample(cfg, cores, prebuilt=pre)
        if i >= args.warmup:
            times.append(dt)
            rates.append(rate)
    value = sum(rates) / len(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "sample": "bounded oracle sample (see cpu_baseline)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- GPU leg
def roofline_report(prof, dgemm_tf, peaks, traffic_file):
    """Top kernel functions by device time in the timed region (per-class CUDA
    events on the library's stream), achieved convention rate vs the measured
    DGEMM peak and the nominal FP64 peak (alu) or the measured HBM copy peak
    (hbm), and the ncu DRAM bytes per launch vs the algorithmic ones."""
    hbm = peaks.get("hbm_gbs", 6553.6)
    tj = {}
    if traffic_file:
        try:
            tj = json.load(open(traffic_file)).get("functions", {})
        except Exception:
            tj = {}
    total_ms = sum(v["ms"] for k, v in prof.items() if k in CLASS_FUNCTION)
    rows = []
    for k, (fn, bound) in CLASS_FUNCTION.items():
        p = prof.get(k)
        if not p or not p["launches"] or p["ms"] <= 0:
            continue
        sec = p["ms"] * 1e-3
        if bound == "hbm":
            achieved = p["bytes"] / sec / 1e9
            peak, unit = hbm, "GB/s"
            frac_nom = achieved / hbm
        else:
            achieved = p["flops"] / sec / 1e12
            peak, unit = dgemm_tf or NOMINAL_FP64_TFLOPS, "TFLOP/s"
            frac_nom = achieved / NOMINAL_FP64_TFLOPS
        nc = ncu_function(tj, NCU_NAME.get(k, ""))
        algo_per_launch = p["bytes"] / p["launches"] if p["bytes"] else None
        rows.append({"class": k, "kernel": fn, "bound": bound, "ms": round(p["ms"], 3),
                     "share": round(p["ms"] / total_ms, 4) if total_ms else None, "launches": p["launches"],
                     "achieved": achieved, "peak": peak, "unit": unit, "frac": achieved / peak if peak else None,
                     "frac_nominal": frac_nom, "gflop": p["flops"] / 1e9, "gb_algorithmic": p["bytes"] / 1e9,
                     "ncu_dram_bytes_per_launch": nc.get("dram_bytes_per_launch"),
                     "algorithmic_bytes_per_launch": algo_per_launch})
    rows.sort(key=lambda r: -r["ms"])
    return rows


def standalone_flush(hm, ctx, torch, dev, X, Y, G, eps, top=3):
    """SURVEY §8(d) config 4 standalone batched flush.  (1) Captured in situ:
    one extra (untimed) product records every level's TRUNC batch; the `top`
    levels by convention flops keep their stacked factors on the device and
    are replayed alone (CUDA events around the TRUNC batch only); the replay
    must reproduce the in-situ ranks.  (2) Synthetic: the captured shape list
    of the largest level, every stack filled with prescribed singular values
    sigma_i = 10^(-i/2) on random orthonormal bases split into 1-8 terms
    (seed [1703, 9085, 4, level]), through hm_test_trunc_batched."""
    import numpy as np
    hm.flush_capture(ctx, 0)
    Z = G.clone()
    hm.addmul(1.0, X, Y, Z, eps)
    Z.free()
    info = hm.flush_capture_info(ctx)
    log(f"flush capture: {len(info)} level batches")
    fl = [sum(trunc_flops(int(a), int(b), int(c), int(d)) for a, b, c, d in zip(L["m"], L["n"], L["l"], L["k"]))
          for L in info]
    order = sorted(range(len(info)), key=lambda i: -fl[i])[:top]
    mask = 0
    for i in order:
        mask |= 1 << i
    hm.flush_capture(ctx, mask)
    Z = G.clone()
    hm.addmul(1.0, X, Y, Z, eps)
    Z.free()
    levels = []
    tot_fl = tot_ms = 0.0
    for i in sorted(order):
        ms, rs = hm.flush_replay(ctx, i, eps, reps=3)
        L = info[i]
        ok = rs == int(L["k"].sum())
        levels.append({"batch": i, "truncations": len(L["m"]), "gflop": fl[i] / 1e9, "ms": ms,
                       "gflops": fl[i] / (ms * 1e-3) / 1e9, "sum_l": int(L["l"].sum()),
                       "max_m": int(max(L["m"].max(), L["n"].max())), "max_l": int(L["l"].max()),
                       "ranks_reproduced": ok})
        tot_fl += fl[i]
        tot_ms += ms
    hm.flush_capture_free(ctx)
    log("flush replay done")
    out = {"captured": {"levels": levels, "gflops": tot_fl / (tot_ms * 1e-3) / 1e9 if tot_ms else None,
                        "all_level_gflop": sum(fl) / 1e9,
                        "note": "TRUNC batches of the top levels by convention flops, replayed from captured stacks"}}
    # synthetic prescribed-sigma stacks on the largest level's shapes (sampled)
    big = order[0]
    L = info[big]
    rng = np.random.default_rng([1703, 9085, 4, big])
    idx = rng.choice(len(L["m"]), size=min(2048, len(L["m"])), replace=False)
    stacks = []
    for j in idx:
        m, n, l = int(L["m"][j]), int(L["n"][j]), int(L["l"][j])
        q = max(1, min(m, n, l) // 2)
        s = 10.0 ** (-np.arange(q) / 2.0)
        U, _ = np.linalg.qr(rng.standard_normal((m, q)))
        V, _ = np.linalg.qr(rng.standard_normal((n, q)))
        nt = int(rng.integers(1, 9))
        cuts = np.sort(rng.choice(np.arange(1, q), size=min(nt - 1, q - 1), replace=False)) if q > 1 else []
        As, Bs = [], []
        for blk in np.split(np.arange(q), cuts):
            As.append(U[:, blk] * s[blk])
            Bs.append(V[:, blk])
        A, B = np.hstack(As), np.hstack(Bs)
        pad = l - A.shape[1]                      # widen to the captured stack width with exact zero columns
        if pad > 0:
            A = np.hstack([A, np.zeros((m, pad))])
            B = np.hstack([B, np.zeros((n, pad))])
        stacks.append((A, B))
    sfl = sum(trunc_flops(a.shape[0], b.shape[0], a.shape[1], 0) for a, b in stacks)
    hm.test_trunc_batched(ctx, stacks, eps)          # warm-up
    # device time of the batched TRUNC only (the upload happens before e0)
    _, ranks, _, ms = hm.test_trunc_batched(ctx, stacks, eps, timed=True)
    out["synthetic"] = {"level_batch": big, "stacks": len(stacks), "gflop": sfl / 1e9, "ms": ms,
                        "gflops": sfl / (ms * 1e-3) / 1e9, "seed": [1703, 9085, 4, int(big)],
                        "recipe": "sigma_i = 10^(-i/2), q = min(m,n,l)/2, random orthonormal bases, 1-8 terms, "
                                  "zero columns up to the captured width l"}
    return out


def run_ours(args, cfg):
    import numpy as np
    import torch

    ws, rank, local = dist_env()
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl")
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    import paper_1703_09085_b200 as hm
    from hm_inputs import sphere_points

    stream = torch.cuda.current_stream(dev)
    ctx = hm.Context(local, stream)
    x, w = sphere_points(cfg["level"])
    t0 = time.time()
    G = ctx.build(x, w, cfg["leaf"], cfg["eta"], cfg["eps"])
    build_s = time.time() - t0
    log(f"built n={len(w)} in {build_s:.1f}s")
    gstats = G.stats()
    X, Y = G.clone(), G.clone()
    nsteps = args.warmup + args.steps
    # fresh Z per step (Z is overwritten); all resident before timing
    Zs = [G.clone() for _ in range(nsteps)]

    def step(i):
        hm.addmul(1.0, X, Y, Zs[i], cfg["eps"])
        Zs[i].free()     # the product is consumed; its memory returns to the pool

    for i in range(args.warmup):
        step(i)
    st = ctx.last_stats()
    flops = st["flops_trunc"] + st["flops_eval"] + st["flops_dense"]
    ctx.profile(True)
    ctx.profile_reset()
    l0 = ctx.last_stats()["kernel_launches"]
    if ws > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize(dev)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev1 = torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.warmup, nsteps):
            step(i)
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    ms = ev0.elapsed_time(ev1)
    log(f"timed {args.steps} steps: {ms / args.steps:.1f} ms/step")
    launches = ctx.last_stats()["kernel_launches"] - l0
    prof = ctx.profile_get()
    ctx.profile(False)
    ms = max_over_ranks(ms, dev)
    ms_step = ms / args.steps
    value = whole_job_value(ws, flops, ms_step)
    # per-class times are summed over the timed steps: per step
    prof_step = {k: {kk: (vv / args.steps if kk in ("ms", "flops", "bytes", "launches") else vv)
                     for kk, vv in v.items()} for k, v in prof.items()}

    # ---- end to end through the C-ABI with host buffers
    dX, dY, dZ = X.export(), Y.export(), G.export()

    def pinned(a):
        t = torch.empty(a.shape, dtype=torch.float64, pin_memory=True)
        t.numpy()[...] = a
        return t.numpy()

    for d_ in (dX, dY, dZ):   # the step's inputs live in pinned host memory
        d_["factors"] = pinned(d_["factors"])
        d_["dense"] = pinned(d_["dense"])
    h2d = sum(int(d["factors"].nbytes + d["dense"].nbytes) for d in (dX, dY, dZ))
    e2e_steps = max(1, min(args.steps, 2))
    # the result is read back into preallocated pinned buffers (sized by one
    # untimed round trip; allocating page-locked memory is not part of a step)
    Xh, Yh, Zh = ctx.import_desc(dX), ctx.import_desc(dY), ctx.import_desc(dZ)
    hm.addmul(1.0, Xh, Yh, Zh, cfg["eps"])
    nf0, nd0 = Zh.export_sizes()
    for m_ in (Xh, Yh, Zh):
        m_.free()
    obufs = (pinned(np.zeros(int(nf0 * 1.1) + 16)), pinned(np.zeros(nd0 + 16)))
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(e2e_steps):
        Xh, Yh, Zh = ctx.import_desc(dX), ctx.import_desc(dY), ctx.import_desc(dZ)
        hm.addmul(1.0, Xh, Yh, Zh, cfg["eps"])
        out = Zh.export(bufs=obufs)
        d2h = int(out["factors"].nbytes + out["dense"].nbytes)
        for m_ in (Xh, Yh, Zh):
            m_.free()
    torch.cuda.synchronize(dev)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_value = ws * flops / (e2e_ms * 1e-3) / 1e9
    log(f"e2e {e2e_ms:.1f} ms/step")

    # ---- roofline of the top kernel functions
    peaks = load_peaks()
    dgemm = measure_dgemm_tflops(torch, dev) if rank == 0 else None
    tfiles = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_traffic.json"))
    traffic_file = os.path.join(ROOT, "profiles", tfiles[-1]) if tfiles else None
    rows = roofline_report(prof_step, dgemm, peaks, traffic_file)
    top = rows[0] if rows else {}
    algo = top.get("gflop", 0) * 1e9 / max(top.get("launches", 1), 1) if top.get("bound") == "alu" else \
        top.get("gb_algorithmic", 0) * 1e9 / max(top.get("launches", 1), 1)
    roof = {"bound": top.get("bound"), "kernel": top.get("kernel"), "achieved": top.get("achieved"),
            "peak": top.get("peak"), "unit": top.get("unit"), "frac": top.get("frac"),
            "frac_nominal": top.get("frac_nominal"),
            "traffic": top.get("ncu_dram_bytes_per_launch"),
            "traffic_source": (f"{os.path.relpath(traffic_file, ROOT)} (ncu dram__bytes_read+write per launch, "
                               f"function {NCU_NAME.get(top.get('class'), '?')})") if traffic_file else None,
            "algorithmic_per_launch": algo, "per_launch_ms": top.get("ms", 0) / max(top.get("launches", 1), 1),
            "launches_per_step": top.get("launches"), "share_of_step": top.get("share"),
            "peak_source": ("measured cuBLAS DGEMM 8192^3 on this box (FP64 has no tcgen05 kind: DMMA/DFMA "
                            f"nominal {NOMINAL_FP64_TFLOPS:.1f} TFLOP/s)") if top.get("bound") == "alu"
            else "MEASURED_PEAKS.json hbm_gbs (copy)",
            "dgemm_cublas_tflops_measured": dgemm, "nominal_fp64_tflops": NOMINAL_FP64_TFLOPS,
            "top_functions": rows[:3],
            "classes": {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                            "gflop": round(v["flops"] / 1e9, 3), "gb": round(v["bytes"] / 1e9, 3)}
                        for k, v in prof_step.items() if v["launches"]}}

    # ---- standalone batched flush (captured + synthetic)
    flush = None
    log("roofline done")
    if rank == 0 and not args.no_flush:
        try:
            flush = standalone_flush(hm, ctx, torch, dev, X, Y, G, cfg["eps"])
        except Exception as e:   # reported, never fatal for the main line
            flush = {"error": repr(e)}

    s0 = None
    # ---- H-LR / H-Cholesky setup seconds (BASELINE configs[1], [2], [4] and the
    # metric's n = 81920 H-LR, "config 4'"), device time with CUDA events
    factor = {}
    log("standalone flush done")
    if rank == 0 and not args.no_factor:
        X.free(), Y.free(), G.free()
        for key, L, leaf, eps, kern, op, reps in FACTOR_RUNS:
            if cfg["level"] < 6 and L > 5:
                continue
            xf, wf = sphere_points(L)
            if L >= 7:
                ctx.trim()   # the n = 327680 build needs the workspaces the earlier legs left behind
            tb = time.time()
            G0 = ctx.build(xf, wf, leaf, 2.0, eps, kernel=kern)
            tb = time.time() - tb
            times = []
            for r in range(reps):
                Gf = G0.clone()
                torch.cuda.synchronize(dev)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                (hm.lr if op == "lr" else hm.chol)(Gf, eps)
                e1.record(stream)
                torch.cuda.synchronize(dev)
                times.append(e0.elapsed_time(e1) / 1e3)
                fst = ctx.last_stats()
                Gf.free()
            G0.free()
            fgf = (fst["flops_trunc"] + fst["flops_eval"] + fst["flops_dense"]) / 1e9
            log(f"{key}: build {tb:.1f}s, setup {min(times):.2f}s")
            factor[key] = {"setup_s": min(times), "runs": len(times), "n": len(wf), "leaf": leaf, "eps": eps,
                           "truncations": fst["truncations"], "trunc_cols": fst["trunc_cols"],
                           "convention_gflop": fgf, "gflops": fgf / min(times), "min_pivot": fst["min_pivot"],
                           "build_s": tb}

    # ---- standard (immediate-update, S0) product next to the accumulated one:
    # the paper's central comparison (Fig. 9).  The
    # device S0 evaluates every term up front into one pool, which does not
    # fit one GPU at config 4 (n = 81920), so both products run on the
    # n = 20480 member of the same family (leaf, eta, eps of config 4) -- last
    # on the device, reported, never fatal.
    if rank == 0 and not args.no_s0:
        try:
            xs, wsf = sphere_points(5 if cfg["level"] >= 6 else cfg["level"])
            Gs = ctx.build(xs, wsf, cfg["leaf"], cfg["eta"], cfg["eps"])
            Xs, Ys = Gs.clone(), Gs.clone()
            res = {}
            for name, fn in (("s2", hm.addmul), ("s0", hm.addmul_std), ("s2", hm.addmul), ("s0", hm.addmul_std)):
                Zs = Gs.clone()
                torch.cuda.synchronize(dev)
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(stream)
                fn(1.0, Xs, Ys, Zs, cfg["eps"])
                e1.record(stream)
                torch.cuda.synchronize(dev)
                sst = ctx.last_stats()
                Zs.free()
                res[name] = (e0.elapsed_time(e1) / 1e3, sst["truncations"], sst["trunc_cols"])
            Xs.free(), Ys.free(), Gs.free()
            s0 = {"n": len(wsf), "leaf": cfg["leaf"], "eps": cfg["eps"],
                  "s0_seconds": res["s0"][0], "s2_seconds": res["s2"][0], "s0_over_s2": res["s0"][0] / res["s2"][0],
                  "s0_truncations": res["s0"][1], "s2_truncations": res["s2"][1],
                  "s0_trunc_cols": res["s0"][2], "s2_trunc_cols": res["s2"][2],
                  "note": "hm_addmul_std (standard algorithm, one truncation per update) vs hm_addmul "
                          "(accumulated updates), second run of each; paper: factor 2-3 (P:L1672-1675)"}
            log(f"S0 {res['s0'][0]:.2f}s / S2 {res['s2'][0]:.2f}s at n={len(wsf)}")
        except Exception as e:
            s0 = {"error": repr(e)}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        rate, dt, sample, gf, _ = oracle_sample(cfg, cores)
        log(f"cpu baseline: {sample}")
        cpu = {"value": rate, "unit": "GFLOP/s", "cores": cores, "kind": "oracle", "sample": sample}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["name"], "n": int(gstats["n"]), "leaf": cfg["leaf"], "eta": cfg["eta"],
                       "eps": cfg["eps"], "parallelism": f"replicas{ws}" if ws > 1 else "single-gpu",
                       "l2": "inputs larger than L2 (X, Y, Z resident, fresh Z clone per step)"},
            "setup_s_per_product": ms_step / 1e3,
            "gflop_per_step": flops / 1e9,
            "truncations": st["truncations"], "trunc_cols": st["trunc_cols"],
            "addproduct_calls": st["addproduct_calls"], "merges": st["merges"],
            "hmatrix": {"blocks": gstats["nblocks"], "adm": gstats["nadm"], "dense": gstats["ndense"],
                        "mean_rank": gstats["mean_rank"], "max_rank": gstats["max_rank"], "build_s": build_s},
            "roofline": roof,
            "hlr_hchol_setup": factor,
            "standalone_flush": flush,
            "s0_vs_s2": s0,
            "cpu_baseline": cpu,
            "e2e": {"value": e2e_value, "unit": "GFLOP/s", "ms_per_step": e2e_ms, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h},
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        print(json.dumps(line))
    if ws > 1:
        torch.distributed.barrier()
        torch.distributed.destroy_process_group()
    return 0


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-factor", action="store_true", help="skip the H-LR / H-Cholesky setup timings")
    ap.add_argument("--no-flush", action="store_true", help="skip the standalone batched-flush timing")
    ap.add_argument("--no-s0", action="store_true", help="skip the standard (S0) product comparison")
    args = ap.parse_args()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # replicas only (the path does not shard): spawn one rank per GPU
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", str(free_port()), os.path.abspath(__file__)] + sys.argv[1:]
        return subprocess.call(cmd)
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
