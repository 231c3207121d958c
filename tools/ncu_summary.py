"""Summarise an ncu report: key metrics, stall reasons, hottest SASS lines.
usage: python tools/ncu_summary.py REPORT.ncu-rep [top_n]"""
import csv, io, subprocess, sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, r = rows[0], rows[2]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum"]
for k in keys:
    if k in hdr:
        print(f"{k:70s} {r[hdr.index(k)]} {rows[1][hdr.index(k)]}")
st = [(h, float(v)) for h, v in zip(hdr, r) if h.startswith("smsp__average_warps_issue_stalled_") and
      h.endswith("_per_issue_active.ratio") and v not in ("", "n/a")]
st.sort(key=lambda t: -t[1])
print("stalls/issue:", ", ".join(f"{h[34:-23]}={v:.2f}" for h, v in st[:8]))
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
tot = sum(float(x[iw] or 0) for x in d2)
print(f"samples {tot:.0f}, sass lines {len(d2)}")
for x in sorted(d2, key=lambda x: -float(x[iw] or 0))[:top]:
    print(x[0][-5:], x[iw].rjust(6), x[ie].rjust(9), x[isrc][:100])
