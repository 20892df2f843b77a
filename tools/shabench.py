"""Cycles per SHA-256 block of the chain engine variants (cg_dbg_sha_bench):
compression alone vs the f64-streaming fast run, per code shape."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_15757_b200 import Context  # noqa: E402

ctx = Context(0)
f = ctx.L.cg_dbg_sha_bench
names = {0: "compress unrolled", 1: "compress rolled", 2: "chain loop0 (2x unrolled)",
         3: "chain loop1 (rolled)", 4: "chain loop2 (1x unrolled)",
         5: "chain rolled fma1 (adds)", 6: "chain rolled fma2 (+shr)",
         7: "chain rolled fma3 (+rotr)"}
for extra, tag in ((0, "1 warp"), (16, "4 warps")):
    for mode in range(5):
        d = C.c_double()
        rc = f(ctx.h, mode | extra, C.c_uint64(20000), C.byref(d))
        print(f"{tag:8s} {names[mode]:28s} {d.value:8.1f} cycles/block rc={rc}", flush=True)
