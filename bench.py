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

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config 4|1] [--no-cpu-baseline]

`--impl reference` times the CPU oracle (oracle/, the reference arm of this
tier) on a bounded sample of the same workload; it is test infrastructure,
never on the product path.
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
]
# profile class -> kernel (for the ncu traffic lookup)
CLASS_KERNEL = {"eval": "k_eval2", "apply_q": "k_applyq", "copy": "k_copy", "memset": None,
                "trunc_fused": "k_trunc_small", "gemm_M": "k_gemm", "dense_add": "k_gemm",
                "qr_blk384": "k_qr_blocked<256, 2, 4, 1>", "qr_blk768": "k_qr_blocked<256, 2, 4, 0>", "qr_blk1536": "k_qr_blocked<512, 1, 4, 0>",
                "svd_smem26k": "k_svd", "svd_global": "k_svd", "svd_smem8k": "k_svd", "svd_smem3k": "k_svd"}
NOMINAL_FP64_TFLOPS = 148 * 64 * 2 * 1.965e9 / 1e12   # DFMA: SMs x FMA/clk x 2 x max clock


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


# ---------------------------------------------------------------- CPU leg
def oracle_sample(cfg, seconds_hint=20.0):
    """The oracle (as it stands) on a bounded sample of the same workload:
    the S2 accumulated product on the level-4 icosphere (n = 5120) with the
    config's leaf size, eta and eps.  Returns (GFLOP/s, seconds, sample text,
    convention GFLOP)."""
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    from hm_inputs import sphere_points
    from oracle.hmatrix import Problem, build
    from oracle.lowrank import TruncCtx
    from oracle.product import addmul_s2
    from oracle.flops import ConventionCounter

    L = min(cfg["level"], 4)
    x, w = sphere_points(L)
    P = Problem(x, w, cfg["leaf"], cfg["eta"])
    G = build(P, cfg["eps"])
    X, Y, Z = G.clone(), G.clone(), G.clone()
    cc = ConventionCounter()
    t0 = time.perf_counter()
    addmul_s2(1.0, X, Y, Z, cfg["eps"], ctx=TruncCtx(cfg["eps"], log_near=False), counter=cc)
    dt = time.perf_counter() - t0
    gf = cc.total_flops() / 1e9
    sample = (f"oracle S2 product (oracle/product.py addmul_s2, NumPy/OpenBLAS, 1 thread) on the n={P.ct.n} "
              f"icosphere (L={L}) with leaf {cfg['leaf']}, eta {cfg['eta']}, eps {cfg['eps']:g}: "
              f"{gf:.2f} convention GFLOP in {dt:.1f} s")
    return gf / dt, dt, sample, gf


def run_reference(args, cfg):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    times, rates = [], []
    sample = ""
    for i in range(args.warmup + args.steps):
        rate, dt, sample, gf = oracle_sample(cfg)
        if i >= args.warmup:
            times.append(dt)
            rates.append(rate)
    value = sum(rates) / len(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GFLOP/s", "n_gpus": ws,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sum(times) / len(times),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg["name"], "sample": "bounded oracle sample (see cpu_baseline)"},
        "cpu_baseline": {"value": value, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample},
        "e2e": {"value": value, "unit": "GFLOP/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------- GPU leg
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
    launches = ctx.last_stats()["kernel_launches"] - l0
    prof = ctx.profile_get()
    ctx.profile(False)
    ms = max_over_ranks(ms, dev)
    ms_step = ms / args.steps
    value = whole_job_value(ws, flops, ms_step)

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
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    d2h = 0
    for _ in range(e2e_steps):
        Xh, Yh, Zh = ctx.import_desc(dX), ctx.import_desc(dY), ctx.import_desc(dZ)
        hm.addmul(1.0, Xh, Yh, Zh, cfg["eps"])
        out = Zh.export()
        d2h = int(out["factors"].nbytes + out["dense"].nbytes)
        for m_ in (Xh, Yh, Zh):
            m_.free()
    torch.cuda.synchronize(dev)
    e2e_ms = (time.perf_counter() - t0) * 1e3 / e2e_steps
    e2e_value = ws * flops / (e2e_ms * 1e-3) / 1e9

    # ---- roofline of the dominant kernel class
    peaks = load_peaks()
    dgemm = measure_dgemm_tflops(torch, dev) if rank == 0 else None
    # dominant single kernel class ("qr" / "jacobi_svd" are aggregates of the bucketed launches)
    top = max(((k, v) for k, v in prof.items() if k not in ("qr", "jacobi_svd")), key=lambda kv: kv[1]["ms"])
    name, p = top
    hbm = peaks.get("hbm_gbs", 6553.6)
    if name in ("eval", "copy", "memset", "apply_q"):
        bound, unit = "hbm", "GB/s"
        achieved = p["bytes"] / (p["ms"] * 1e-3) / 1e9 if p["ms"] else 0.0
        peak = hbm
        peak_src = "MEASURED_PEAKS.json hbm_gbs (copy)"
    else:
        bound, unit = "alu", "TFLOP/s"
        achieved = p["flops"] / (p["ms"] * 1e-3) / 1e12 if p["ms"] else 0.0
        peak = NOMINAL_FP64_TFLOPS
        peak_src = "FP64 DFMA nominal 148 SM x 64 FMA/clk x 2 x 1.965 GHz (DESIGN.md §6); tcgen05 has no f64 kind"
    # dram traffic per launch of the class's kernel: the committed ncu launch
    # list of one bench step (scripts/ncu_traffic.py -> profiles/*_traffic.json)
    traffic, traffic_src = None, None
    kern = CLASS_KERNEL.get(name)
    tfiles = sorted(f for f in os.listdir(os.path.join(ROOT, "profiles")) if f.endswith("_traffic.json"))
    if kern and tfiles:
        try:
            tj = json.load(open(os.path.join(ROOT, "profiles", tfiles[-1])))
            if kern in tj["kernels"]:
                traffic = tj["kernels"][kern]["dram_bytes_per_launch"]
                traffic_src = f"profiles/{tfiles[-1]} ({kern}, ncu dram__bytes_read+write per launch)"
        except Exception:
            pass
    roof = {"bound": bound, "kernel": name, "achieved": achieved, "peak": peak, "unit": unit,
            "frac": achieved / peak if peak else None, "traffic": traffic, "traffic_source": traffic_src,
            "algorithmic_per_launch": (p["bytes"] if bound == "hbm" else p["flops"]) / max(p["launches"], 1),
            "per_launch_ms": p["ms"] / max(p["launches"], 1), "launches": p["launches"], "peak_source": peak_src,
            "dgemm_cublas_tflops_measured": dgemm,
            "classes": {k: {"ms": round(v["ms"], 3), "launches": v["launches"],
                            "gflop": round(v["flops"] / 1e9, 3), "gb": round(v["bytes"] / 1e9, 3)}
                        for k, v in prof.items() if v["launches"]}}

    # ---- H-LR / H-Cholesky setup seconds (BASELINE configs[1], [2] and the
    # metric's n = 81920 H-LR, "config 4'"), device time with CUDA events
    factor = {}
    if rank == 0 and not args.no_factor:
        for key, L, leaf, eps, kern, op, reps in FACTOR_RUNS:
            xf, wf = sphere_points(L)
            G0 = ctx.build(xf, wf, leaf, 2.0, eps, kernel=kern)
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
            factor[key] = {"setup_s": min(times), "runs": len(times), "n": len(wf), "leaf": leaf, "eps": eps,
                           "truncations": fst["truncations"], "min_pivot": fst["min_pivot"]}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        rate, dt, sample, gf = oracle_sample(cfg)
        cpu = {"value": rate, "unit": "GFLOP/s", "cores": 1, "kind": "oracle", "sample": sample}

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


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-factor", action="store_true", help="skip the H-LR / H-Cholesky setup timings")
    args = ap.parse_args()
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
