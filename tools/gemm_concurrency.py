"""Weight-gradient (64 output tiles on 74 CTA pairs) and activation-gradient products of
one MLP layer back to back on one stream vs on two streams (CUDA events on both)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402

M, h = 16384, 1024
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()  # noqa: E731
x, dmid, w1 = r(M, h), r(M, 4 * h), r(h, 4 * h)
g1 = torch.zeros(h, 4 * h, device="cuda")
dx = torch.empty(M, h, device="cuda")
s2 = torch.cuda.Stream()


def dw():
    K.gemm(x.t(), dmid, g1, c=g1, alpha=-1e-4)


def dxp():
    K.gemm(dmid, w1.t(), dx)


def serial():
    dw()
    dxp()


def concurrent():
    cur = torch.cuda.current_stream()
    s2.wait_stream(cur)
    with torch.cuda.stream(s2):
        dw()
    dxp()
    cur.wait_stream(s2)


for name, fn in (("dW1 alone", dw), ("dx_fc1 alone", dxp), ("serial", serial), ("two streams", concurrent),
                 ("serial", serial), ("two streams", concurrent)):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        fn()
    e1.record()
    torch.cuda.synchronize()
    print(f"{name:14s} {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us", flush=True)
