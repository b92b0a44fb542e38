"""The BERT-large 1x1 training step's GEMMs in isolation, with their epilogues,
vs cuBLAS (torch.matmul, same output dtype). SG_GEMM_BN forces the N tile."""
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


def main():
    dev = "cuda"
    M, h = 16384, 1024
    bf, f32 = torch.bfloat16, torch.float32
    r = lambda *s: torch.randn(*s, device=dev).to(bf)  # noqa: E731
    x, w_qkv, w_d, w1, w2 = r(M, h), r(h, 3 * h), r(h, h), r(h, 4 * h), r(4 * h, h)
    bias3, bias1, bias4 = (torch.randn(n, device=dev) for n in (3 * h, h, 4 * h))
    ctx, act, dy = r(M, h), r(M, 4 * h), r(M, h)
    resid = torch.randn(M, h, device=dev)
    o_qkv = torch.empty(M, 3 * h, device=dev, dtype=bf)
    o_h32 = torch.empty(M, h, device=dev)
    o_h16 = torch.empty(M, h, device=dev, dtype=bf)
    o_4h = torch.empty(M, 4 * h, device=dev, dtype=bf)
    mid = torch.empty(M, 4 * h, device=dev, dtype=bf)
    g_qkv = torch.empty(h, 3 * h, device=dev)
    g_d = torch.empty(h, h, device=dev)
    g_1 = torch.empty(h, 4 * h, device=dev)
    dqkv, dmid = r(M, 3 * h), r(M, 4 * h)
    cases = [
        ("qkv fwd  x@Wqkv+b ->bf16", lambda: K.gemm(x, w_qkv, o_qkv, bias=bias3), (x, w_qkv, o_qkv)),
        ("dense fwd ctx@Wd+b+res ->f32", lambda: K.gemm(ctx, w_d, o_h32, bias=bias1, c=resid), (ctx, w_d, o_h32)),
        ("fc1 fwd  +b gelu ->bf16,mid", lambda: K.gemm(x, w1, o_4h, bias=bias4, act=K.ACT_GELU, aux=mid), (x, w1, o_4h)),
        ("fc2 fwd  act@W2+b+res ->f32", lambda: K.gemm(act, w2, o_h32, bias=bias1, c=resid), (act, w2, o_h32)),
        ("dmid  dy@W2^T ->bf16", lambda: K.gemm(dy, w2.t(), o_4h), (dy, w2.t(), o_4h)),
        ("dx fc1 dmid@W1^T ->f32", lambda: K.gemm(dmid, w1.t(), o_h32), (dmid, w1.t(), o_h32)),
        ("dctx dy@Wd^T ->bf16", lambda: K.gemm(dy, w_d.t(), o_h16), (dy, w_d.t(), o_h16)),
        ("dx qkv dqkv@Wqkv^T ->f32", lambda: K.gemm(dqkv, w_qkv.t(), o_h32), (dqkv, w_qkv.t(), o_h32)),
        ("dW1 x^T@dmid ->f32", lambda: K.gemm(x.t(), dmid, g_1), (x.t(), dmid, g_1)),
        ("dW2 act^T@dy ->f32", lambda: K.gemm(act.t(), dy, g_1.view(4 * h, h)), (act.t(), dy, g_1.view(4 * h, h))),
        ("dWqkv x^T@dqkv ->f32", lambda: K.gemm(x.t(), dqkv, g_qkv), (x.t(), dqkv, g_qkv)),
        ("dWd ctx^T@dy ->f32", lambda: K.gemm(ctx.t(), dy, g_d), (ctx.t(), dy, g_d)),
    ]
    for name, fn, (a, b, o) in cases:
        m, k = a.shape
        n = b.shape[1]
        fl = 2.0 * m * n * k
        us = bench(fn)
        ref = bench(lambda: torch.matmul(a, b, out=o) if o.dtype == bf else torch.matmul(a, b).float())
        print(f"{name:32s} M={m:5d} N={n:5d} K={k:5d}  sg {us:7.1f} us {fl / us / 1e6:7.1f} TF/s | "
              f"cublas {ref:7.1f} us {fl / ref / 1e6:7.1f} TF/s", flush=True)


if __name__ == "__main__":
    main()
