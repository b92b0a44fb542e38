"""Phase timeline of the flash backward (instrumented build from tools/trace_build.py: libsg_trace.so with
sg_debug_ftrace): CTA 0, softmax warp 4 lane 0 (buffer 0) and the MMA thread (buffer 1)."""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ["SG_LIB_PATH"] = "paper_2104_05343_b200/libsg_trace.so"
sys.path.insert(0, ".")
from paper_2104_05343_b200 import _lib, kernels as K  # noqa: E402

b, s, nh, d = 32, 512, 16, 64
hb = nh * d
qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
dout = torch.randn(b * s, hb, device="cuda").bfloat16()
out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, nh, s, device="cuda")
drow = torch.empty(b, nh, s, device="cuda")
dq = torch.zeros(b * s, hb, device="cuda")
dqkv = torch.empty(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
K.attn_rowdot(dout, out, nh, d, s, drow)
for _ in range(3):
    K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv)
torch.cuda.synchronize()
buf = np.zeros((2, 8192), dtype=np.uint64)
lib = _lib.lib()
lib.sg_debug_ftrace.argtypes = [ctypes.c_void_p]
assert lib.sg_debug_ftrace(buf.ctypes.data) == 0
for w in range(2):
    ev = (buf[w] >> np.uint64(56)).astype(int)
    t = (buf[w] & np.uint64(0xffffffffffffff)).astype(np.int64)
    n = int(np.count_nonzero(buf[w]))
    ev, t = ev[:n], t[:n]
    # mean gap from each event to the next, by event id
    gaps = {}
    for k in range(n - 1):
        gaps.setdefault(ev[k], []).append(t[k + 1] - t[k])
    print("buffer", w, "events", n, "span", t[-1] - t[0] if n else 0)
    for e_ in sorted(gaps):
        g = np.array(gaps[e_])
        print(f"  after ev {e_:2d}: mean {g.mean():7.0f} clk  median {np.median(g):7.0f}  n={len(g)}")
