"""Phase timeline of a flash kernel from the instrumented build (tools/trace_build.py:
libsg_trace.so, SG_TR stamps, sg_debug_trace): CTA 0, per buffer the mean / median
clocks from each event to the next.

    python tools/ftrace.py fwd|bwd [b s nh d]
"""
import ctypes
import os
import sys

import numpy as np
import torch

os.environ.setdefault("SG_LIB_PATH", "paper_2104_05343_b200/libsg_trace.so")
sys.path.insert(0, ".")
from paper_2104_05343_b200 import _lib, kernels as K  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "fwd"
b, s, nh, d = (int(x) for x in sys.argv[2:6]) if len(sys.argv) >= 6 else (32, 512, 16, 64)
hb = nh * d
qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
dout = torch.randn(b * s, hb, device="cuda").bfloat16()
out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, nh, s, device="cuda")
drow = torch.empty(b, nh, s, device="cuda")
dq = torch.zeros(b * s, hb, device="cuda")
dqkv = torch.empty(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
lib = _lib.lib()
lib.sg_debug_trace.argtypes = [ctypes.c_void_p]
K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
K.attn_rowdot(dout, out, nh, d, s, drow)
torch.cuda.synchronize()
for _ in range(3):
    lib.sg_debug_trace_clear()
    if which == "fwd":
        K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
    else:
        K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv)
    torch.cuda.synchronize()
buf = np.zeros((4, 8192), dtype=np.uint64)
assert lib.sg_debug_trace(buf.ctypes.data) == 0
for w in range(4):
    ev = (buf[w] >> np.uint64(56)).astype(int)
    t = (buf[w] & np.uint64(0xffffffffffffff)).astype(np.int64)
    n = int(np.count_nonzero(buf[w]))
    if n == 0:
        continue
    ev, t = ev[:n], t[:n]
    gaps = {}
    for k in range(n - 1):
        gaps.setdefault((ev[k], ev[k + 1]), []).append(t[k + 1] - t[k])
    print(f"buffer {w}: events {n}, span {t[-1] - t[0]} clk")
    for key in sorted(gaps):
        g = np.array(gaps[key])
        print(f"  {key[0]:2d} -> {key[1]:2d}: mean {g.mean():7.0f}  median {np.median(g):7.0f}  n={len(g)}")

# absolute timeline (same SM clock for every buffer): events of blocks [G0, G0 + 3)
if os.environ.get("SG_FTRACE_TIMELINE"):
    G0 = int(os.environ["SG_FTRACE_TIMELINE"])
    rows = []
    for w in range(4):
        n = int(np.count_nonzero(buf[w]))
        ev = (buf[w][:n] >> np.uint64(56)).astype(int)
        t = (buf[w][:n] & np.uint64(0xffffffffffffff)).astype(np.int64)
        blk = np.cumsum(ev == 0) - 1  # event 0 opens a block
        for k in range(n):
            if G0 <= blk[k] < G0 + 3:
                rows.append((int(t[k]), w, int(blk[k]), int(ev[k])))
    rows.sort()
    t0 = rows[0][0] if rows else 0
    for t, w, g, e in rows:
        print(f"{t - t0:7d}  buf{w} G{g} ev{e}")
