"""Per-kernel DRAM traffic from an ncu launch list taken with
`--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum`
(one bench step, scripts/ncu_step.py).  Writes a JSON summary that bench.py
reads for `roofline.traffic` (dram bytes per launch of the dominant kernel).

    python scripts/ncu_traffic.py LAUNCHES.csv OUT.json
"""
import collections
import csv
import json
import sys

SCALE_T = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
SCALE_B = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}


def main(path, out):
    rows = list(csv.reader(open(path)))
    i = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    hdr, data = rows[i], rows[i + 1:]
    ki, ni, ui, vi, ii = (hdr.index(k) for k in ("Kernel Name", "Metric Name", "Metric Unit", "Metric Value", "ID"))
    per = collections.defaultdict(dict)
    names = {}
    for r in data:
        if len(r) <= vi:
            continue
        v = float(r[vi].replace(",", ""))
        unit, metric = r[ui], r[ni]
        if metric == "gpu__time_duration.sum":
            v *= SCALE_T.get(unit, 1.0)
        else:
            v *= SCALE_B.get(unit, 1.0)
        per[r[ii]][metric] = v
        names[r[ii]] = r[ki].split("(")[0].replace("hm::", "").replace("void ", "")
    agg = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    for lid, m in per.items():
        a = agg[names[lid]]
        a["launches"] += 1
        a["ms"] += m.get("gpu__time_duration.sum", 0.0)
        a["dram_bytes"] += m.get("dram__bytes_read.sum", 0.0) + m.get("dram__bytes_write.sum", 0.0)
    tot = sum(a["ms"] for a in agg.values())
    res = {}
    for k, a in sorted(agg.items(), key=lambda kv: -kv[1]["ms"]):
        res[k] = {"launches": a["launches"], "ms": round(a["ms"], 3), "share": round(a["ms"] / tot, 4),
                  "dram_bytes_per_launch": a["dram_bytes"] / a["launches"],
                  "dram_gbs": a["dram_bytes"] / (a["ms"] * 1e-3) / 1e9 if a["ms"] else None}
    # aggregated by kernel FUNCTION (template instantiations / buckets merged)
    fun = collections.defaultdict(lambda: {"launches": 0, "ms": 0.0, "dram_bytes": 0.0})
    for k, a in agg.items():
        f = fun[k.split("<")[0].strip()]
        for key in ("launches", "ms", "dram_bytes"):
            f[key] += a[key]
    fres = {k: {"launches": a["launches"], "ms": round(a["ms"], 3), "share": round(a["ms"] / tot, 4),
                "dram_bytes_per_launch": a["dram_bytes"] / a["launches"], "dram_bytes": a["dram_bytes"]}
            for k, a in sorted(fun.items(), key=lambda kv: -kv[1]["ms"])}
    json.dump({"source": path, "total_ms": tot, "kernels": res, "functions": fres}, open(out, "w"), indent=1)
    for k, a in res.items():
        print(f"{k:20s} {a['launches']:5d} {a['ms']:10.1f} ms {100 * a['share']:5.1f}%  "
              f"{a['dram_bytes_per_launch'] / 1e6:10.1f} MB/launch  {a['dram_gbs'] or 0:8.0f} GB/s")


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
