import sys
import torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402
torch.manual_seed(0)
M, h = 16384, 1024
dy = torch.randn(M, h, device="cuda").bfloat16()
w2 = torch.randn(4 * h, h, device="cuda").bfloat16()
mid = torch.randn(M, 4 * h, device="cuda").bfloat16()
out = torch.empty(M, 4 * h, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    K.gemm(dy, w2.t(), out, act=K.ACT_DGELU, aux=mid)
torch.cuda.synchronize()
