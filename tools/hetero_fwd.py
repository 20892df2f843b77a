"""Forward-only timing of each C3 model (R50 / R101 / VGG-16 / MBv2, one
replica each, batch B) and its GEMM share. Dev tool:
  python tools/hetero_fwd.py [B] [arch] [iters]   (arch: one model only)"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context, Model, lib  # noqa: E402
from paper_2205_15757_b200.workload import hetero_group  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ONLY = sys.argv[2] if len(sys.argv) > 2 else None
ITERS = int(sys.argv[3]) if len(sys.argv) > 3 else 10
ctx = Context(0)
L = lib()
L.cg_model_flops_per_input.restype = C.c_double
out = hetero_group()
files, digs = out[0], out[1]
tot = 0.0
for arch, f, d in zip(("resnet50", "resnet101", "vgg16", "mobilenet_v2"), files, digs):
    if ONLY and arch != ONLY:
        continue
    m = Model.load_cnn(ctx, f, d)
    flops = L.cg_model_flops_per_input(m.h) * B
    ms = C.c_double()
    assert L.cg_dbg_forward_bench(ctx.h, m.h, B, ITERS, C.byref(ms)) == 0, L.cg_last_error(ctx.h)
    L.cg_timing_enable(1)
    ms2 = C.c_double()
    L.cg_dbg_forward_bench(ctx.h, m.h, B, 3, C.byref(ms2))
    t, n = C.c_double(), C.c_uint64()
    L.cg_timing_read(0, C.byref(t), C.byref(n))
    a, na = C.c_double(), C.c_uint64()
    L.cg_timing_read(3, C.byref(a), C.byref(na))
    L.cg_timing_enable(0)
    tot += ms.value
    print(f"{arch:13s} B={B}: {ms.value:7.3f} ms/fwd  {flops / ms.value / 1e9:7.1f} TFLOP/s  "
          f"gemm {t.value / 4:.3f} ms ({n.value // 4} launches)  aux {a.value / 4:.3f} ms")
print(f"sum of forwards {tot:.3f} ms per {B}-request batch")
