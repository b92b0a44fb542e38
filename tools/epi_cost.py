"""Epilogue cost per output tile: the step's epilogue variants at tiny K (the
mainloop is negligible, so time ~ epilogue + HBM traffic).

    python tools/epi_cost.py [K] [case-prefix]
"""
import sys

import torch

sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def t(fn, n=30):
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


def main():
    kk = int(sys.argv[1]) if len(sys.argv) > 1 else 64
    only = sys.argv[2] if len(sys.argv) > 2 else None  # run one case 4x (ncu target)
    M, N = 16384, 4096
    bf = torch.bfloat16
    a = torch.randn(M, kk, device="cuda").to(bf)
    b = torch.randn(kk, N, device="cuda").to(bf)
    o16 = torch.empty(M, N, device="cuda", dtype=bf)
    o32 = torch.empty(M, N, device="cuda")
    aux = torch.randn(M, N, device="cuda").to(bf)
    c32 = torch.randn(M, N, device="cuda")
    bias = torch.randn(N, device="cuda")
    cs = torch.zeros(N, device="cuda")
    tiles = (M // 256) * (N // 256)
    cases = [
        ("bf16 out", lambda: K.gemm(a, b, o16), 2),
        ("f32 out", lambda: K.gemm(a, b, o32), 4),
        ("bf16 +bias", lambda: K.gemm(a, b, o16, bias=bias), 2),
        ("bf16 +colsum", lambda: K.gemm(a, b, o16, colsum=cs), 2),
        ("dgelu (aux in)", lambda: K.gemm(a, b, o16, act=K.ACT_DGELU, aux=aux), 4),
        ("gelu+aux out", lambda: K.gemm(a, b, o16, bias=bias, act=K.ACT_GELU, aux=aux), 4),
        ("f32 +C f32", lambda: K.gemm(a, b, o32, c=c32), 8),
    ]
    for name, fn, bpe in cases:
        if only is not None:
            if name.startswith(only):
                for _ in range(4):
                    fn()
                torch.cuda.synchronize()
            continue
        us = t(fn)
        gb = M * N * bpe / us / 1e3
        print(f"{name:16s} K={kk:4d} {us:7.1f} us  {us * 1e3 / (tiles / 74):6.0f} ns/tile/pair  "
              f"{gb:6.0f} GB/s epilogue IO", flush=True)


if __name__ == "__main__":
    main()
