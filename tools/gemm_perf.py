"""Quick tcgen05 GEMM throughput check vs cuBLAS (torch.matmul) on one GPU."""
import sys
import time

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels  # noqa: E402


def bench(fn, iters=20, warm=5):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


def main():
    torch.manual_seed(0)
    shapes = [(8192, 8192, 8192, "ab"), (8192, 8192, 8192, "abt"), (8192, 8192, 8192, "atb"),
              (16384, 3072, 1024, "ab"), (16384, 1024, 4096, "ab"), (16384, 1024, 3072, "abt"),
              (1024, 3072, 16384, "atb"), (4096, 4096, 4096, "ab")]
    for M, N, K, lay in shapes:
        a = torch.randn(M, K, device="cuda").bfloat16() if lay != "atb" else torch.randn(K, M, device="cuda").bfloat16().t()
        b = torch.randn(K, N, device="cuda").bfloat16() if lay != "abt" else torch.randn(N, K, device="cuda").bfloat16().t()
        out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        t_sg = bench(lambda: kernels.gemm(a, b, out))
        t_cb = bench(lambda: torch.matmul(a, b, out=out))
        fl = 2.0 * M * N * K
        print(f"{lay:4s} M={M} N={N} K={K}: sg {t_sg*1e3:8.1f} us {fl/t_sg/1e9:7.1f} TF/s | cublas {t_cb*1e3:8.1f} us {fl/t_cb/1e9:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
