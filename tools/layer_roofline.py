"""Per-launch roofline of one ResNet-50 replica forward (B images).

Joins an ncu launch list (gpu__time_duration.sum, cold-cache serialized) with
the algorithmic FLOPs and compulsory HBM bytes of each launch, in the order
CnnModel::forward launches them (csrc/cnn.cu plan_for). floor = max(FLOPs /
peak_flops, bytes / peak_bw) with the measured peaks (MEASURED_PEAKS.json).

  python tools/layer_roofline.py <launches.csv> [B]
"""
import csv
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def plan(B=128, S=224):
    """(name, flops, hbm_bytes) per launch, same order as plan_for."""
    L = []
    H1, H2 = S // 2, S // 4
    px = lambda h: B * h * h  # noqa: E731
    # conv1 on the im2col operand (K=192 padded, 147 real)
    L.append(("conv1 7x7/2", 2 * px(H1) * 64 * 147, px(H1) * 192 * 2 + px(H1) * 64 * 2))
    L.append(("maxpool", 0, px(H1) * 64 * 2 + px(H2) * 64 * 2))
    H, cin = H2, 64
    for stage, (w, n) in enumerate(((64, 3), (128, 4), (256, 6), (512, 3))):
        for i in range(n):
            s = 2 if (i == 0 and stage > 0) else 1
            Ho = H // s
            cout = 4 * w
            L.append((f"l{stage + 1}.{i} c1 1x1 {cin}->{w}", 2 * px(H) * cin * w,
                      px(H) * cin * 2 + B * (H + 2) ** 2 * w * 2))
            if s == 1:
                L.append((f"l{stage + 1}.{i} c2 3x3 {w}", 2 * px(Ho) * 9 * w * w,
                          B * (H + 2) ** 2 * w * 2 + px(Ho) * w * 2))
            else:
                L.append((f"l{stage + 1}.{i} gather3x3/2", 0,
                          B * (H + 2) ** 2 * w * 2 + px(Ho) * 9 * w * 2))
                L.append((f"l{stage + 1}.{i} c2 3x3/2 {w}", 2 * px(Ho) * 9 * w * w,
                          px(Ho) * 9 * w * 2 + px(Ho) * w * 2))
            if i == 0:
                if s == 2:
                    L.append((f"l{stage + 1}.{i} gather1x1/2", 0,
                              px(H) * cin * 2 + px(Ho) * cin * 2))
                L.append((f"l{stage + 1}.{i} ds 1x1 {cin}->{cout}", 2 * px(Ho) * cin * cout,
                          px(Ho) * cin * 2 + px(Ho) * cout * 2))
            L.append((f"l{stage + 1}.{i} c3 1x1 {w}->{cout} +res", 2 * px(Ho) * w * cout,
                      px(Ho) * w * 2 + 2 * px(Ho) * cout * 2))
            H, cin = Ho, cout
    L.append(("avgpool", 0, px(H) * cin * 2 + B * cin * 2))
    L.append(("fc", 2 * B * cin * 1000, B * cin * 2 + 1000 * cin * 2 + B * 1000 * 4))
    return L


def main():
    path = sys.argv[1]
    B = int(sys.argv[2]) if len(sys.argv) > 2 else 128
    pk = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    bw, fl = pk["hbm_gbs"] * 1e9, pk["bf16_tflops"] * 1e12
    rows = list(csv.reader(open(path)))
    hdr = next(r for r in rows if "Kernel Name" in r)
    data = [dict(zip(hdr, r)) for r in rows if len(r) == len(hdr) and r != hdr]
    idx = [i for i, d in enumerate(data)
           if "conv1_im2col" in d["Kernel Name"] or "chw_to_s2d16" in d["Kernel Name"]]
    seg = [d for d in data[idx[-1] + 1:]]
    P = plan(B)
    if len(seg) != len(P):
        print(f"launch count {len(seg)} != plan {len(P)}; partial join")
    tot_t = tot_f = 0.0
    print(f"{'launch':34s} {'us':>8s} {'floor':>8s} {'eff':>6s} {'TFLOP/s':>8s} {'TB/s':>6s}")
    for (name, f, b), d in zip(P, seg):
        t = float(d["Metric Value"].replace(",", "")) / 1e3  # us
        floor = max(f / fl, b / bw) * 1e6
        tot_t += t
        tot_f += floor
        print(f"{name:34s} {t:8.1f} {floor:8.1f} {floor / t:6.2f} {f / t / 1e6:8.1f} {b / t / 1e6:6.2f}")
    print(f"{'TOTAL':34s} {tot_t:8.1f} {tot_f:8.1f} {tot_f / tot_t:6.2f}")


if __name__ == "__main__":
    main()
