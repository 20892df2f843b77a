"""Summarise a chrome trace written by `bench.py --trace`: per-stream busy
time, the main stream's idle gaps (and which kernels bracket them), and the
top kernels by total device time.

  python tools/timeline.py gpurun_out/trace.json [--gap-us 5]
"""
import argparse
import collections
import json


def short(name, n=60):
    name = name.replace("void ", "")
    return name if len(name) <= n else name[:n] + "..."


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("trace")
    ap.add_argument("--gap-us", type=float, default=5.0)
    ap.add_argument("--top", type=int, default=25)
    a = ap.parse_args()
    ev = json.load(open(a.trace))["traceEvents"]
    ks = [e for e in ev if e.get("ph") == "X" and e.get("cat") in ("kernel", "gpu_memcpy", "gpu_memset")]
    by_stream = collections.defaultdict(list)
    for e in ks:
        by_stream[e["args"].get("stream", e.get("tid"))].append(e)
    t0 = min(e["ts"] for e in ks)
    t1 = max(e["ts"] + e["dur"] for e in ks)
    print(f"window {1e-3 * (t1 - t0):.3f} ms, {len(ks)} device ops")
    main_stream = max(by_stream, key=lambda s: sum(e["dur"] for e in by_stream[s]))
    for s, L in sorted(by_stream.items(), key=lambda kv: -sum(e["dur"] for e in kv[1])):
        busy = sum(e["dur"] for e in L)
        print(f"stream {s}: {len(L)} ops, busy {1e-3 * busy:.3f} ms"
              f"{'  <- main' if s == main_stream else ''}")
    L = sorted(by_stream[main_stream], key=lambda e: e["ts"])
    gaps = []
    for x, y in zip(L, L[1:]):
        g = y["ts"] - (x["ts"] + x["dur"])
        if g > a.gap_us:
            gaps.append((g, short(x["name"], 45), short(y["name"], 45)))
    tot = sum(g for g, _, _ in gaps)
    print(f"main-stream gaps > {a.gap_us} us: {len(gaps)}, total {1e-3 * tot:.3f} ms")
    agg = collections.defaultdict(lambda: [0.0, 0])
    for g, x, y in gaps:
        agg[(x, y)][0] += g
        agg[(x, y)][1] += 1
    for (x, y), (g, n) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:12]:
        print(f"  {1e-3 * g:8.3f} ms  x{n:<4d} after {x}  before {y}")
    kt = collections.defaultdict(lambda: [0.0, 0])
    for e in ks:
        kt[short(e["name"], 90)][0] += e["dur"]
        kt[short(e["name"], 90)][1] += 1
    print("top device ops (all streams):")
    for n, (d, c) in sorted(kt.items(), key=lambda kv: -kv[1][0])[:a.top]:
        print(f"  {1e-3 * d:9.3f} ms  x{c:<5d} {n}")


if __name__ == "__main__":
    main()
