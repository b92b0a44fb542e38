"""Time the dAct-shaped ABT GEMM with each epilogue feature toggled."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


torch.manual_seed(0)
M, h = 16384, 1024
dy = torch.randn(M, h, device="cuda").bfloat16()
w2 = torch.randn(4 * h, h, device="cuda").bfloat16()
mid = torch.randn(M, 4 * h, device="cuda").bfloat16()
out = torch.empty(M, 4 * h, device="cuda", dtype=torch.bfloat16)
out32 = torch.empty(M, 4 * h, device="cuda")
cs = torch.zeros(4 * h, device="cuda")
c32 = torch.randn(M, 4 * h, device="cuda")
print("plain bf16   ", t(lambda: K.gemm(dy, w2.t(), out)))
print("plain fp32   ", t(lambda: K.gemm(dy, w2.t(), out32)))
print("+colsum      ", t(lambda: K.gemm(dy, w2.t(), out, colsum=cs)))
print("+dgelu       ", t(lambda: K.gemm(dy, w2.t(), out, act=K.ACT_DGELU, aux=mid)))
print("+dgelu+cs    ", t(lambda: K.gemm(dy, w2.t(), out, act=K.ACT_DGELU, aux=mid, colsum=cs)))
print("+C fp32      ", t(lambda: K.gemm(dy, w2.t(), out32, c=c32)))
print("gelu fwd     ", t(lambda: K.gemm(dy, w2.t(), out, act=K.ACT_GELU, aux=mid)))
