"""Summarise an ncu --page source --csv dump: top SASS instructions by warp-stall samples per kernel.
usage: ncu -i rep --page source --csv --print-source sass > x.csv; python tools/ncu_src.py x.csv <kernel-substr> [N]"""
import csv
import sys

path, pat = sys.argv[1], sys.argv[2]
N = int(sys.argv[3]) if len(sys.argv) > 3 else 40
cur, hdr, rows = None, None, []
for r in csv.reader(open(path)):
    if r and r[0] == "Kernel Name":
        cur = r[1]
        hdr = None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and cur and pat in cur:
        rows.append(dict(zip(hdr, r)))
tot = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows)
print("kernel samples:", tot, "instructions:", len(rows))
stall_cols = [c for c in (hdr or []) if c.startswith("stall_") and "Not Issued" not in c]
top = sorted(rows, key=lambda x: -int(x["Warp Stall Sampling (All Samples)"] or 0))[:N]
for x in top:
    s = int(x["Warp Stall Sampling (All Samples)"] or 0)
    st = sorted(((c, int(x[c] or 0)) for c in stall_cols), key=lambda y: -y[1])[:3]
    print(f"{s:6d} {100*s/max(tot,1):5.1f}% {x['Address'][-5:]} {x['Source'].strip()[:60]:60s} {st}")
