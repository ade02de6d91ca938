"""Markdown summary of a bench.py JSON line (for DESIGN.md).  Usage: python scripts/bench_table.py BENCH.json"""
import json
import sys
d = json.load(open(sys.argv[1]))
r = d["roofline"]
print(f"| product n = 81920 (config 4), device time / step | {d['ms_per_step'] / 1e3:.3f} s |")
print(f"| convention FP64 rate of the product | {d['value']:.0f} GFLOP/s = {d['value'] / 1e3 / r['peak']:.3f} of the measured DGEMM ({r['peak']:.1f} TF/s) |")
print(f"| e2e (host descriptions in, result out) | {d['e2e']['ms_per_step'] / 1e3:.3f} s ({d['e2e']['value']:.0f} GFLOP/s) |")
for t in r["top_functions"]:
    print(f"| `{t['kernel']}` | {t['ms']:.0f} ms, share {t['share']:.2f}, {t['achieved']:.2f} {t['unit']} = {t['frac']:.3f} of peak |")
for k, v in r["classes"].items():
    if k in ("trunc_fused", "apply_q", "copy", "gemm_M", "tsqr_stack", "memset"):
        print(f"| class `{k}` | {v['ms']:.0f} ms |")
for k, v in d["hlr_hchol_setup"].items():
    print(f"| {k} | {v['setup_s']:.2f} s ({v.get('gflops', 0):.0f} convention GFLOP/s, {v['truncations']} truncations) |")
sf = d["standalone_flush"]
print(f"| standalone flush, captured top-3 levels | {sf['captured']['gflops']:.0f} GFLOP/s |")
print(f"| standalone flush, synthetic | {sf['synthetic']['gflops']:.0f} GFLOP/s |")
if "s0_vs_s2" in d and d["s0_vs_s2"]:
    print("| S0 vs S2 |", json.dumps(d["s0_vs_s2"]), "|")
cb = d["cpu_baseline"]
print(f"| CPU oracle ({cb['cores']} cores) | {cb['value']:.0f} GFLOP/s |")
