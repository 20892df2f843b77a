"""Text summary of one kernel in an `ncu --set full --import-source on`
report: duration, SOL, DRAM bytes, tensor-pipe activity, warp-stall reasons
and the CUDA source lines holding the most stall samples. Dev tool:
  python tools/ncu_summary.py report.ncu-rep [title]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
title = sys.argv[2] if len(sys.argv) > 2 else rep


def ncu(*args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


raw = list(csv.reader(io.StringIO(ncu("--page", "raw", "--csv"))))
d = dict(zip(raw[0], raw[2]))
print(f"# {title}")
print(f"kernel: {d.get('Kernel Name', '?')[:120]}")
keys = [("gpu__time_duration.sum", "duration (us)"),
        ("dram__bytes_read.sum", "DRAM read (MB)"), ("dram__bytes_write.sum", "DRAM write (MB)"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "memory SOL %"),
        ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM SOL %"),
        ("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "tensor pipe active %"),
        ("lts__t_sectors.avg.pct_of_peak_sustained_elapsed", "L2 sectors %"),
        ("sm__inst_executed.avg.per_cycle_active", "IPC (per SM)"),
        ("launch__registers_per_thread", "registers/thread"),
        ("launch__grid_size", "grid")]
for k, label in keys:
    if k in d:
        print(f"{label:24s} {d[k]}")
st = {k[len('smsp__pcsamp_warps_issue_stalled_'):]: float(v) for k, v in d.items()
      if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
      and v.replace(".", "", 1).isdigit()}
tot = sum(st.values()) or 1.0
print("warp-stall samples: " + ", ".join(f"{k} {v / tot * 100:.1f}%"
                                          for k, v in sorted(st.items(), key=lambda t: -t[1])[:8]))
src = list(csv.reader(io.StringIO(ncu("--page", "source", "--csv", "--print-source", "cuda,sass"))))
hdr = next((r for r in src if "Warp Stall Sampling (All Samples)" in r), None)
if hdr:
    i_s = hdr.index("Warp Stall Sampling (All Samples)")
    rows = [r for r in src if len(r) == len(hdr) and r[2] == "-" and r[0].isdigit()]
    t = sum(float(r[i_s] or 0) for r in rows) or 1.0
    print("top source lines by stall samples (gemm_sm100.cu line: share):")
    for r in sorted(rows, key=lambda r: -float(r[i_s] or 0))[:12]:
        print(f"  L{r[0]:>5s} {float(r[i_s]) / t * 100:5.1f}%  {r[1].strip()[:90]}")
