import ctypes as C, sys
sys.path.insert(0,'.')
from paper_2205_15757_b200 import Context
ctx=Context(0)
f=ctx.L.cg_dbg_sha_bench
for mode in (0,1):
    for nb in (1000, 20000):
        d=C.c_double()
        rc=f(ctx.h, mode, C.c_uint64(nb), C.byref(d)); print("mode",mode,"nblocks",nb,"cycles/block",d.value, rc)
