"""Forward-only timing of one ResNet-50 replica (no SHA concurrency) plus
per-class kernel attribution. Dev tool: python tools/fwd_bench.py [B]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context, Model, lib  # noqa: E402
from paper_2205_15757_b200.workload import resnet_group  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 128
ctx = Context(0)
files, digs, _ = resnet_group("resnet50", replicas=1)
m = Model.load_cnn(ctx, files[0], digs[0])
L = lib()
L.cg_model_flops_per_input.restype = C.c_double
flops = L.cg_model_flops_per_input(m.h) * B
ms = C.c_double()
assert L.cg_dbg_forward_bench(ctx.h, m.h, B, 10, C.byref(ms)) == 0, L.cg_last_error(ctx.h)
print(f"forward B={B}: {ms.value:.3f} ms  {flops / ms.value / 1e9:.1f} TFLOP/s (algorithmic)")
L.cg_timing_enable(1)
L.cg_dbg_forward_bench(ctx.h, m.h, B, 3, C.byref(ms))
t, n = C.c_double(), C.c_uint64()
L.cg_timing_read(0, C.byref(t), C.byref(n))
print(f"  timed pass {ms.value:.3f} ms/fwd; gemm {t.value / 4:.3f} ms/fwd over {n.value // 4} launches")
L.cg_timing_enable(0)
