"""One step GEMM shape in isolation (ncu target): python tools/gemm_one.py {dmid|dmidg|dW1|fc1|qkv|dense} [reps]."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402

M, h = 16384, 1024
dev = "cuda"
bf = torch.bfloat16
r = lambda *s: torch.randn(*s, device=dev).to(bf)  # noqa: E731
which = sys.argv[1] if len(sys.argv) > 1 else "dmid"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
if which == "dmid":
    a, b, o = r(M, h), r(4 * h, h).t(), torch.empty(M, 4 * h, device=dev, dtype=bf)
    fn = lambda: K.gemm(a, b, o)  # noqa: E731
elif which == "dmidg":
    a, b, o = r(M, h), r(4 * h, h).t(), torch.empty(M, 4 * h, device=dev, dtype=bf)
    aux, cs = r(M, 4 * h), torch.zeros(4 * h, device=dev)
    fn = lambda: K.gemm(a, b, o, act=K.ACT_DGELU, aux=aux, colsum=cs)  # noqa: E731
elif which == "dW1":  # weight gradient x^T dmid (both operands MN-major), the step's top GEMM
    a, b, o = r(M, h).t(), r(M, 4 * h), torch.empty(h, 4 * h, device=dev)
    fn = lambda: K.gemm(a, b, o)  # noqa: E731
elif which == "fc1":
    a, b, o = r(M, h), r(h, 4 * h), torch.empty(M, 4 * h, device=dev, dtype=bf)
    mid, bias = torch.empty_like(o), torch.randn(4 * h, device=dev)
    fn = lambda: K.gemm(a, b, o, bias=bias, act=K.ACT_GELU, aux=mid)  # noqa: E731
elif which == "qkv":
    a, b, o = r(M, h), r(h, 3 * h), torch.empty(M, 3 * h, device=dev, dtype=bf)
    bias = torch.randn(3 * h, device=dev)
    fn = lambda: K.gemm(a, b, o, bias=bias)  # noqa: E731
else:
    a, b, o = r(M, h), r(h, h), torch.empty(M, h, device=dev)
    bias, res = torch.randn(h, device=dev), torch.randn(M, h, device=dev)
    fn = lambda: K.gemm(a, b, o, bias=bias, c=res)  # noqa: E731
for _ in range(reps):
    fn()
torch.cuda.synchronize()
