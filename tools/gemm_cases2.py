"""The step's epilogue-heavy GEMMs in isolation (ncu target): dAct with GELU'
+ column sums, and the fused attention softmax product."""
import math
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def main():
    torch.manual_seed(0)
    dev = "cuda"
    M, h = 16384, 1024
    dy = torch.randn(M, h, device=dev).bfloat16()
    w2 = torch.randn(4 * h, h, device=dev).bfloat16()
    mid = torch.randn(M, 4 * h, device=dev).bfloat16()
    dmid = torch.empty(M, 4 * h, device=dev, dtype=torch.bfloat16)
    cs = torch.zeros(4 * h, device=dev)
    b, n, s, d = 32, 16, 512, 64
    q = torch.randn(b, n, s, d, device=dev).bfloat16()
    k = torch.randn(b, n, s, d, device=dev).bfloat16()
    p = torch.empty(b, n, s, s, device=dev, dtype=torch.bfloat16)
    reps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    for _ in range(reps):
        K.gemm(dy, w2.t(), dmid, act=K.ACT_DGELU, aux=mid, colsum=cs)
        K.gemm(q, k.transpose(-1, -2), p, alpha=1 / math.sqrt(d), mode=K.EPI_SOFTMAX)
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(10):
        K.gemm(dy, w2.t(), dmid, act=K.ACT_DGELU, aux=mid, colsum=cs)
    ev[1].record()
    for _ in range(10):
        K.gemm(q, k.transpose(-1, -2), p, alpha=1 / math.sqrt(d), mode=K.EPI_SOFTMAX)
    ev[2].record()
    torch.cuda.synchronize()
    print(f"dAct+GELU'+colsum: {ev[0].elapsed_time(ev[1]) / 10 * 1e3:.1f} us;  QK^T+softmax: {ev[1].elapsed_time(ev[2]) / 10 * 1e3:.1f} us")


if __name__ == "__main__":
    main()
