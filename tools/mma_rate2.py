"""Cycles per K=16 SS-mode MMA (M=128, 148 CTAs) for N = 64 / 128: the same
A/B tiles every MMA vs rotating over distinct tiles (as a real mainloop
reads), with one or two accumulators. Dev tool."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
for N in (64, 128):
    for mode, label in ((0, "same tiles, 1 acc "), (1, "same tiles, 2 accs"),
                        (3, "rotating,   1 acc "), (4, "rotating,   2 accs")):
        c = C.c_double()
        rc = ctx.L.cg_dbg_mma_rate(ctx.h, N, 4096, 148, mode, C.byref(c))
        assert rc == 0, ctx.L.cg_last_error(ctx.h)
        print(f"N={N:3d} {label}: {c.value:6.1f} cycles/MMA")
c = C.c_double()
assert ctx.L.cg_dbg_mma_rate(ctx.h, 64, 4096, 148, 5, C.byref(c)) == 0, ctx.L.cg_last_error(ctx.h)
print(f"N= 64 s2d stem pattern (SW32, K = 16 rows, row-shifted A, 16 tap tiles): {c.value:6.1f} cycles/MMA")
