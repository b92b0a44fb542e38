"""One flash forward + backward launch at a given shape (ncu target).

    python tools/flash_one.py b s nh d
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402

b, s, nh, d = (int(x) for x in sys.argv[1:5])
hb = nh * d
qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
dout = torch.randn(b * s, hb, device="cuda").bfloat16()
out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(b, nh, s, device="cuda")
drow = torch.empty(b, nh, s, device="cuda")
dq = torch.zeros(b * s, hb, device="cuda")
dqkv = torch.empty(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
for _ in range(2):
    K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
    K.attn_rowdot(dout, out, nh, d, s, drow)
    K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv)
torch.cuda.synchronize()
