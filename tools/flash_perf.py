"""Time the flash attention kernels (CUDA events, warm, back to back) for given shapes.

    python tools/flash_perf.py [b,s,nh,d ...]     default: the BERT and GPT (1x1, 2x4) shapes
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def timeit(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def run(b, s, nh, d):
    hb = nh * d
    qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
    dout = torch.randn(b * s, hb, device="cuda").bfloat16()
    out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, nh, s, device="cuda")
    drow = torch.empty(b, nh, s, device="cuda")
    dq = torch.zeros(b * s, hb, device="cuda")
    dqkv = torch.empty(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
    fl = 4.0 * b * nh * s * s * d  # forward: QK^T and PV
    tf = timeit(lambda: K.flash_attn_fwd(qkv, b, s, nh, d, out, lse))
    tb = timeit(lambda: K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv))
    tr = timeit(lambda: K.attn_rowdot(dout, out, nh, d, s, drow))
    print(f"b={b} s={s} nh={nh} d={d}: fwd {tf*1e3:.1f} us {fl/tf/1e9:.0f} TF/s | "
          f"bwd {tb*1e3:.1f} us {2.5*fl/tb/1e9:.0f} TF/s | rowdot {tr*1e3:.1f} us", flush=True)


shapes = [tuple(int(x) for x in a.split(",")) for a in sys.argv[1:]] or \
    [(32, 512, 16, 64), (4, 2048, 16, 64), (8, 2048, 32, 128), (4, 2048, 8, 128)]
for sh in shapes:
    run(*sh)
