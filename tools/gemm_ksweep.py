"""Per-tile overhead probe: 16384 x N x K plain bf16-out products for a K sweep
(wave count fixed by M x N), plus the fp32-out variant."""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402
from tools.gemm_step_shapes import bench  # noqa: E402


def main():
    M = 16384
    for N in (1024, 4096):
        for Kd in (512, 1024, 2048, 4096, 8192):
            a = torch.randn(M, Kd, device="cuda").bfloat16()
            b = torch.randn(Kd, N, device="cuda").bfloat16()
            for f32 in (False, True):
                o = torch.empty(M, N, device="cuda", dtype=torch.float32 if f32 else torch.bfloat16)
                us = bench(lambda: K.gemm(a, b, o))
                fl = 2.0 * M * N * Kd
                print(f"M={M} N={N:5d} K={Kd:5d} {'f32' if f32 else 'bf16'}: {us:7.1f} us {fl / us / 1e6:7.1f} TF/s",
                      flush=True)


if __name__ == "__main__":
    main()
