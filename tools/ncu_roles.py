"""Per-role summary of a source-level ncu CSV (ncu --page source --csv --print-source sass): the
SASS of a warp-specialised kernel is split into role regions by landmark instructions, and each
region's warp-stall samples, executed warp instructions, top stall reasons and opcode mix are
printed.  usage: ncu_roles.py SASS.csv.gz KERNEL-SUBSTR"""
import collections
import csv
import gzip
import io
import re
import sys

path, pat = sys.argv[1], sys.argv[2]
rows, cur, hdr = [], None, None
for r in csv.reader(io.TextIOWrapper(gzip.open(path)) if path.endswith(".gz") else open(path)):
    if r and r[0] == "Kernel Name":
        cur, hdr = r[1], None
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and cur and pat in cur:
        rows.append(dict(zip(hdr, r)))
stall = [c for c in hdr if c.startswith("stall_") and "Not Issued" not in c]
# role regions: each warpgroup role starts with its setmaxnreg (USETMAXREG); the control
# warpgroup's region is split at its first TMA load / MMA into producer and MMA issuers
sm = [i for i, x in enumerate(rows) if "USETMAXREG" in x["Source"]]
names = {"0x30": "control (producer + MMA issuers)", "0x40": "control (producer + MMA issuers)",
         "0x88": "P/dS epilogue", "0x68": "epilogue", "0x50": "dQ read-out + d pos_bias"}
ends = [("prologue", 0, sm[0] if sm else len(rows))]
for j, i in enumerate(sm):
    nxt = sm[j + 1] if j + 1 < len(sm) else len(rows)
    reg = rows[i]["Source"].strip().split()[-1]
    ends.append((names.get(reg, "role " + reg), i, nxt))
tot_s = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in rows)
print(f"kernel {pat}: {tot_s} warp-stall samples, {len(rows)} SASS lines")
for name, a, b in ends:
    if b <= a:
        continue
    seg = rows[a:b]
    s = sum(int(x["Warp Stall Sampling (All Samples)"] or 0) for x in seg)
    ex = sum(int(x["Instructions Executed"] or 0) for x in seg)
    st = collections.Counter()
    ops = collections.Counter()
    for x in seg:
        for c in stall:
            st[c[6:]] += int(x[c] or 0)
        op = re.sub(r"^@!?U?P\w+\s+", "", x["Source"].strip()).split(" ")[0]
        ops[op] += int(x["Instructions Executed"] or 0)
    print(f"\n{name}: {100 * s / max(tot_s, 1):.0f}% of samples, {ex / 1e6:.0f} M warp instructions")
    print("  stalls:", ", ".join(f"{k} {100 * v / max(s, 1):.0f}%" for k, v in st.most_common(5)))
    print("  opcodes:", ", ".join(f"{k} {100 * v / max(ex, 1):.0f}%" for k, v in ops.most_common(8)))
