"""Stall-reason totals per instruction class: ncu_stalls.py REPORT [exec_count_filter]"""
import csv, io, subprocess, sys, collections
rep = sys.argv[1]; flt = sys.argv[2] if len(sys.argv) > 2 else None
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(src))); hdr = rows[1]
data = [x for x in rows[2:] if len(x) == len(hdr) and x[0] != "Address"]
seen, d2 = set(), []
for x in data:
    if x[0] not in seen:
        seen.add(x[0]); d2.append(x)
ie, isrc = hdr.index("Instructions Executed"), hdr.index("Source")
cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
tot = collections.Counter(); byop = collections.defaultdict(collections.Counter)
for x in d2:
    if flt and x[ie] != flt: continue
    op = (x[isrc].split()[1] if x[isrc].startswith("@") else x[isrc].split()[0]) if x[isrc] else "?"
    for i in cols:
        v = float(x[i] or 0)
        tot[hdr[i]] += v; byop[op][hdr[i]] += v
print("total:", ", ".join(f"{k[6:]}={v:.0f}" for k, v in tot.most_common(10)))
for op, c in sorted(byop.items(), key=lambda t: -sum(t[1].values()))[:12]:
    print(f"{op:28s} {sum(c.values()):6.0f}  " + ", ".join(f"{k[6:]}={v:.0f}" for k, v in c.most_common(4)))
