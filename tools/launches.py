"""Summarise an ncu --metrics gpu__time_duration.sum CSV: the last forward
(from the last conv1 operand launch: chw_to_s2d16 / conv1_im2col) with per-launch times. Dev tool."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        # CSVs with several metrics per launch: keep the duration rows
        if d.get("Metric Name", "gpu__time_duration.sum") == "gpu__time_duration.sum":
            data.append(d)
start = sys.argv[2] if len(sys.argv) > 2 and not sys.argv[2].startswith("-") else None
starts = [start] if start else ["chw_to_s2d16", "conv1_im2col"]
idx = [i for i, d in enumerate(data) if any(x in d["Kernel Name"] for x in starts)]
# -p: the last COMPLETE forward (between the last two starts) when the
# capture ends mid-step
seg = (data[idx[-2]:idx[-1]] if "-p" in sys.argv and len(idx) > 1
       else data[idx[-1]:] if idx else data)
tot = 0.0
agg = collections.defaultdict(lambda: [0, 0.0])
for d in seg:
    v = float(d["Metric Value"].replace(",", "")) / 1e3
    tot += v
    n = d["Kernel Name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[-44:]
    agg[n][0] += 1
    agg[n][1] += v
    if "-v" in sys.argv:
        print(f"{n:44s} grid {d['Grid Size']:14s} {v:9.1f} us")
for n, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:44s} x{c:4d} {v:10.1f} us {100 * v / tot:5.1f}%")
print(f"total {tot:.1f} us over {len(seg)} launches")
