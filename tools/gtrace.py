"""Epilogue phase timeline of sg_gemm (instrumented build from tools/trace_build.py: libsg_trace.so with
sg_debug_gtrace): CTA 0 epilogue warp 4 lane 0 (buffer 0), MMA thread (buffer 1).
    python tools/gtrace.py CASE   (CASE as in tools/gemm_one.py)"""
import ctypes
import os
import runpy
import sys

import numpy as np

os.environ["SG_LIB_PATH"] = "paper_2104_05343_b200/libsg_trace.so"
sys.argv = ["gemm_one.py", sys.argv[1], "3"]
runpy.run_path("tools/gemm_one.py")
import torch  # noqa: E402

sys.path.insert(0, ".")
from paper_2104_05343_b200 import _lib  # noqa: E402

torch.cuda.synchronize()
buf = np.zeros((4, 4096), dtype=np.uint64)
lib = _lib.lib()
lib.sg_debug_gtrace.argtypes = [ctypes.c_void_p]
assert lib.sg_debug_gtrace(buf.ctypes.data) == 0
for w in range(2):
    n = int(np.count_nonzero(buf[w]))
    ev = (buf[w][:n] >> np.uint64(56)).astype(int)
    t = (buf[w][:n] & np.uint64(0xffffffffffffff)).astype(np.int64)
    gaps = {}
    for k in range(n - 1):
        gaps.setdefault((ev[k], ev[k + 1]), []).append(t[k + 1] - t[k])
    print("buffer", w, "events", n, "span", (t[-1] - t[0]) if n else 0)
    for key in sorted(gaps):
        g = np.array(gaps[key])
        print(f"  {key[0]:2d}->{key[1]:2d}: mean {g.mean():7.0f}  median {np.median(g):7.0f}  n={len(g)}")
