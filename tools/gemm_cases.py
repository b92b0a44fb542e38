"""Run the training step's main GEMM shapes a few times (target for ncu -k regex:gemm_kernel)."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def main():
    torch.manual_seed(0)
    dev = "cuda"
    M = 16384
    x = torch.randn(M, 1024, device=dev).bfloat16()
    w1 = torch.randn(1024, 4096, device=dev).bfloat16()
    b1 = torch.randn(4096, device=dev)
    mid = torch.empty(M, 4096, device=dev, dtype=torch.bfloat16)
    act = torch.empty(M, 4096, device=dev, dtype=torch.bfloat16)
    w2 = torch.randn(4096, 1024, device=dev).bfloat16()
    out = torch.empty(M, 1024, device=dev)
    res = torch.randn(M, 1024, device=dev)
    for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 3):
        K.gemm(x, w1, act, bias=b1, act=K.ACT_GELU, aux=mid)      # fc1 (GELU epilogue, 2 bf16 outputs)
        K.gemm(act, w2, out, c=res)                                # fc2 (+residual, fp32 out)
        K.gemm(act.t(), x, torch.empty(4096, 1024, device=dev))   # dW (A^T B, both MN-major)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
