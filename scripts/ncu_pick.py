"""From an ncu launch list (gpu__time_duration per launch) pick, for every kernel
instantiation of interest, its LONGEST launch and print one capture spec per
line: `<mangled-name regex>:<tag>:<launch index among that instantiation>`
(read by scripts/gpu_prof.sh for the --set full captures).

    python scripts/ncu_pick.py LAUNCHES.csv [min_share]
"""
import collections
import csv
import re
import sys


def mangled(name):
    m = re.match(r"k_qr_reg<(\d+), (\d+), (\d+)>", name)
    if m:
        return "_ZN2hm8k_qr_regILi%sELi%sELi%sEEE" % m.groups(), "qr_reg_%s_%s_%s" % m.groups()
    m = re.match(r"k_qr_blocked<(\d+), (\d+), (\d+), (\d+)>", name)
    if m:
        return "_ZN2hm12k_qr_blockedILi%sELi%sELi%sELb%sEE" % m.groups(), "qr_blocked_%s" % m.group(1)
    simple = {"k_svd": "_ZN2hm5k_svd", "k_trunc_small": "_ZN2hm13k_trunc_small", "k_eval2": "_ZN2hm7k_eval2",
              "k_applyq_dmma": "_ZN2hm13k_applyq_dmma", "k_gemm2": "_ZN2hm7k_gemm2", "k_qrs_update": "_ZN2hm12k_qrs_update"}
    if name in simple:
        return simple[name], name[2:]
    return None


def main(path, min_share=0.015):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[i], rows[i + 1:]
    ki, ni, vi = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Value"))
    seen = collections.defaultdict(int)
    best, total = {}, collections.defaultdict(float)
    for r in data:
        if len(r) <= vi or r[ni] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("hm::", "").replace("void ", "").strip()
        t = float(r[vi].replace(",", ""))
        idx = seen[name]
        seen[name] += 1
        total[name] += t
        if name not in best or t > best[name][0]:
            best[name] = (t, idx)
    alltime = sum(total.values())
    for name, (t, idx) in sorted(best.items(), key=lambda kv: -total[kv[0]]):
        mg = mangled(name)
        if mg and total[name] >= min_share * alltime:
            print(f"{mg[0]}:{mg[1]}:{idx}")


if __name__ == "__main__":
    main(sys.argv[1], float(sys.argv[2]) if len(sys.argv) > 2 else 0.015)
