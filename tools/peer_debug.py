"""Debug the in-process peer CG (two ranks on one GPU): run, then dump exchange state."""
import sys
import ctypes as C
import numpy as np
sys.path.insert(0, "tests")
sys.path.insert(0, ".")
import torch
import test_gpu_peer as T

x_ref, it_ref, ranks = T._setup(3, 2, (4, 2, 2), 2, seed=7)
print("single-domain iterations", it_ref, flush=True)
try:
    out = T._solve_all(ranks)
    print("ok", [it for _, it in out])
except Exception as e:
    print("FAILED", e)
for r in ranks:
    ex = r["ops"].peer
    buf = (C.c_uint64 * 66)()
    ex._ctx.lib.hx_peer_state(ex._ctx.h, buf)
    print("rank", r["sub"].rank, "seq", buf[0], "err", buf[1], "flags", list(buf[2:4]), flush=True)
