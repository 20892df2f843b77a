"""Per-launch roofline of the conv GEMM launches of one C2 step (3 replicas
grouped per launch, batch B), from an ncu CSV of `-k regex:conv_gemm`
launches with gpu__time_duration.sum, dram__bytes_read.sum and
dram__bytes_write.sum. floor = max(FLOPs / peak, compulsory bytes / peak BW)
with the measured peaks (MEASURED_PEAKS.json); launch order = csrc/cnn.cu
ResNet::ops (conv1, per block c1, c2, c3 (+ the projection shortcut in each
stage's first block), fc).

  python tools/step_roofline.py <ncu.csv> [B] [replicas] [--json traffic.json]

--json writes the step's GEMM DRAM traffic summary that bench.py reports as
roofline.traffic (profiles/r02_gemm_step_traffic.json).
"""
import collections
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SC = {'byte': 1, 'Kbyte': 1e3, 'Mbyte': 1e6, 'Gbyte': 1e9, 'ns': 1e-3, 'nsecond': 1e-3,
      'us': 1, 'usecond': 1, 'ms': 1e3, 'msecond': 1e3}


def plan(B, R, S=224):
    L = []
    px = lambda h: B * h * h  # noqa: E731
    H1, H = S // 2, S // 4
    G = (S + 6) // 2  # s2d stem: 2 planes x 16 B per grid pixel
    L.append(("conv1 7x7/2", 2 * px(H1) * 64 * 147 * R, B * G * G * 32 + R * px(H1) * 64 * 2))
    cin = 64
    for stage, (w, n) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for i in range(n):
            s = 2 if (i == 0 and stage > 0) else 1
            Ho, cout = H // s, 4 * w
            L.append((f"l{stage + 1}.{i} c1 1x1 {cin}->{w}", 2 * px(H) * cin * w * R,
                      R * (px(H) * cin * 2 + px(H) * w * 2)))
            L.append((f"l{stage + 1}.{i} c2 3x3{'/2' if s == 2 else ''} {w}",
                      2 * px(Ho) * 9 * w * w * R, R * (px(H) * w * 2 + px(Ho) * w * 2)))
            if i == 0:  # c3 + projection shortcut fused (K = w + cin)
                L.append((f"l{stage + 1}.{i} c3+ds 1x1 {w}+{cin}->{cout}",
                          2 * px(Ho) * (w + cin) * cout * R,
                          R * (px(Ho) * (w + cin) * 2 + px(Ho) * cout * 2)))
            else:
                L.append((f"l{stage + 1}.{i} c3 1x1 {w}->{cout} +res", 2 * px(Ho) * w * cout * R,
                          R * (px(Ho) * w * 2 + 2 * px(Ho) * cout * 2)))
            H, cin = Ho, cout
    L.append(("fc", 2 * B * cin * 1000 * R, R * (B * cin * 2 + B * 1000 * 4)))
    return L


def main():
    argv = list(sys.argv[1:])
    out_json = None
    if "--json" in argv:
        k = argv.index("--json")
        out_json = argv[k + 1]
        del argv[k:k + 2]
    path = argv[0]
    B = int(argv[1]) if len(argv) > 1 else 128
    R = int(argv[2]) if len(argv) > 2 else 3
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw, fl = pk["hbm_gbs"] * 1e9, pk.get("bf16_tflops_sustained", pk["bf16_tflops"]) * 1e12
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if r and r[0] == "ID"][0]
    ix = {h: i for i, h in enumerate(rows[hi])}
    per = collections.OrderedDict()
    for r in rows[hi + 1:]:
        d = per.setdefault(int(r[ix["ID"]]), {"name": r[ix["Kernel Name"]]})
        d[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", "")) * SC[r[ix["Metric Unit"]]]
    P = plan(B, R)
    # the last complete forward: the len(P) GEMM launches after the last
    # conv1 operand kernel that has them all (chains, trees and auxiliary
    # kernels interleave from other streams and are skipped)
    seq = list(per.values())
    gem = None
    for i in range(len(seq) - 1, -1, -1):
        if "conv1_im2col" in seq[i]["name"] or "chw_to_s2d16" in seq[i]["name"]:
            g = [d for d in seq[i + 1:] if "conv_gemm" in d["name"]][:len(P)]
            if len(g) == len(P):
                gem = g
                break
    per = collections.OrderedDict(enumerate(gem))
    print(f"{'launch':30s} {'us':>7s} {'floor':>7s} {'eff':>5s} {'TFLOP/s':>8s} "
          f"{'DRAM TB/s':>9s} {'traffic/compulsory':>9s}")
    T = F = RD = WR = 0.0
    for (name, f, b), d in zip(P, per.values()):
        RD += d["dram__bytes_read.sum"]
        WR += d["dram__bytes_write.sum"]
        t = d["gpu__time_duration.sum"]
        traffic = d["dram__bytes_read.sum"] + d["dram__bytes_write.sum"]
        floor = max(f / fl, b / bw) * 1e6
        T += t
        F += floor
        print(f"{name:30s} {t:7.1f} {floor:7.1f} {floor / t:5.2f} {f / t / 1e6:8.1f} "
              f"{traffic / t / 1e6:9.2f} {traffic / b:9.2f}")
    print(f"{'TOTAL':30s} {T:7.1f} {F:7.1f} {F / T:5.2f}   (peaks: {fl / 1e12:.0f} TFLOP/s, "
          f"{bw / 1e12:.2f} TB/s)")
    if out_json:
        with open(out_json, "w") as fo:
            json.dump({"launches": len(P), "gemm_us_per_step_ncu": round(T, 1),
                       "dram_read_bytes_per_step": RD, "dram_write_bytes_per_step": WR,
                       "traffic_bytes_per_step": RD + WR,
                       "traffic_bytes_per_launch_avg": (RD + WR) / len(P),
                       "source": "ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
                                 "dram__bytes_write.sum --clock-control none of bench.py --profile: "
                                 f"the {len(P)} conv_gemm launches of one C2 step (3 replicas "
                                 "grouped, final round-2 build), cold-cache serialised "
                                 f"({os.path.relpath(path, ROOT)})"}, fo, indent=1)
            fo.write("\n")


if __name__ == "__main__":
    main()
