"""Summarise an ncu report's source page: stall mix, opcode mix, hottest source lines.
Usage: python scripts/ncu_src.py file.ncu-rep [topN]"""
import csv, subprocess, sys, collections, io
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(txt)))
h = next(i for i, r in enumerate(rows) if r and r[0] == "Address")
hdr = rows[h]; ix = {k: i for i, k in enumerate(hdr)}; data = [r for r in rows[h + 1:] if len(r) == len(hdr)]
S = ix["# Samples"]; N = ix["Instructions Executed"]
tot_s = sum(int(r[S]) for r in data); tot_n = sum(int(r[N]) for r in data)
print("kernel:", rows[0][1] if rows[0] else "?", "| samples", tot_s, "warp-instr", tot_n)
st = [k for k in hdr if k.startswith("stall_") and "Not Issued" not in k]
agg = {k: sum(int(r[ix[k]]) for r in data) for k in st}
print("stalls:", ", ".join(f"{k[6:]} {100*v/tot_s:.0f}%" for k, v in sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
op = collections.Counter(); ops = collections.Counter()
for r in data:
    t = [x for x in r[ix["Source"]].split() if not x.startswith("@")]
    if t: op[t[0].split(".")[0]] += int(r[N]); ops[t[0].split(".")[0]] += int(r[S])
print("opcodes:", ", ".join(f"{k} {100*v/tot_n:.0f}%/{100*ops[k]/tot_s:.0f}%" for k, v in op.most_common(14)), "(instr% / sample%)")
print("hottest instructions:")
for r in sorted(data, key=lambda r: -int(r[S]))[:top]:
    why = max(st, key=lambda k: int(r[ix[k]]))
    print(f"  {100*int(r[S])/tot_s:5.1f}%  {r[ix['Source']].strip()[:70]:70s} {why[6:]}")
