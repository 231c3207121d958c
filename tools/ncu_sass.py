"""Print SASS (with samples / exec counts) around addresses: ncu_sass.py REPORT addr_suffix [before after] ..."""
import csv, io, subprocess, sys
rep = sys.argv[1]
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr = rows[1]
data = [x for x in rows[2:] if len(x) == len(hdr) and x[0] != "Address"]
seen, d2 = set(), []
for x in data:
    if x[0] not in seen:
        seen.add(x[0]); d2.append(x)
iw, ie, isrc = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed"), hdr.index("Source")
args = sys.argv[2:]
b, a = 8, 4
addrs = [x[0][-5:] for x in d2]
for t in args:
    if ":" in t:
        t, b, a = t.split(":"); b, a = int(b), int(a)
    i = addrs.index(t)
    for x in d2[max(0, i - b):i + a]:
        print(x[0][-5:], x[iw].rjust(6), x[ie].rjust(9), x[isrc][:110])
    print("----")
