"""Per-launch table of the last complete forward in an ncu CSV
(gpu__time_duration.sum, dram__bytes_read.sum, dram__bytes_write.sum) of
`tools/hetero_fwd.py B arch 2`: the forward's launch sequence is found as the
repeating tail of the capture. Dev tool:
  python tools/fwd_launches.py <ncu.csv>"""
import collections
import csv
import sys

SC = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-3, 'nsecond': 1e-3,
      'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}
rows = list(csv.reader(open(sys.argv[1])))
hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
ix = {h: i for i, h in enumerate(rows[hi])}
per = collections.OrderedDict()
for r in rows[hi + 1:]:
    d = per.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]]})
    d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * SC[r[ix["Metric Unit"]]]
seq = list(per.values())
names = [d["name"] for d in seq]
P = next(p for p in range(5, len(seq) // 2 + 1) if names[-p:] == names[-2 * p:-p])
tot = 0.0
print(f"{'launch':52s} {'us':>8s} {'DRAM R MB':>10s} {'DRAM W MB':>10s} {'TB/s':>6s}")
for d in seq[-P:]:
    t = d["gpu__time_duration.sum"]
    rd, wr = d["dram__bytes_read.sum"] / 1e6, d["dram__bytes_write.sum"] / 1e6
    tot += t
    n = d["name"].split("(")[0].replace("void ", "").replace("(anonymous namespace)::", "")[-52:]
    print(f"{n:52s} {t:8.1f} {rd:10.1f} {wr:10.1f} {(rd + wr) / t:6.2f}")
print(f"total {tot:.1f} us over {P} launches")
