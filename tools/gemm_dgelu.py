"""dAct GEMM with GELU' (+ b1 column sums) fused in the epilogue vs GEMM + sg_dgelu pass."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def bench(fn, iters=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters * 1e3


M, h = 16384, 1024
dev = "cuda"
dy = torch.randn(M, h, device=dev).bfloat16()
w2 = torch.randn(4 * h, h, device=dev).bfloat16()
mid = torch.randn(M, 4 * h, device=dev).bfloat16()
dmid = torch.empty(M, 4 * h, device=dev, dtype=torch.bfloat16)
cs = torch.zeros(4 * h, device=dev)
fused = bench(lambda: K.gemm(dy, w2.t(), dmid, act=K.ACT_DGELU, aux=mid, colsum=cs))
ref = dmid.clone()
split = bench(lambda: (K.gemm(dy, w2.t(), dmid), K.dgelu(dmid, mid, dmid, cs)))
K.gemm(dy, w2.t(), dmid)
K.dgelu(dmid, mid, dmid, cs)
err = ((dmid.float() - ref.float()).abs().max() / ref.float().abs().max()).item()
print(f"fused GEMM+GELU'+colsum {fused:.1f} us | GEMM then dgelu pass {split:.1f} us | rel diff {err:.2e}")
