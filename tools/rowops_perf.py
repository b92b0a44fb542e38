"""HBM roofline check of the row kernels at the BERT-large 1x1 shapes (CUDA events, GB/s)."""
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
    f32, bf = torch.float32, torch.bfloat16
    dy, x, res = (torch.randn(M, h, device=dev) for _ in range(3))
    dx = torch.empty(M, h, device=dev)
    dx2 = torch.empty(M, h, device=dev, dtype=bf)
    mean, rstd = torch.randn(M, device=dev), torch.rand(M, device=dev) + 0.5
    stats = torch.randn(M, 2, device=dev)
    gamma = torch.randn(h, device=dev)
    beta = torch.randn(h, device=dev)
    dg, db, ds = (torch.zeros(h, device=dev) for _ in range(3))
    y = torch.empty(M, h, device=dev, dtype=bf)
    dact = torch.randn(M, 4 * h, device=dev).to(bf)
    mid = torch.randn(M, 4 * h, device=dev).to(bf)
    cs4 = torch.zeros(4 * h, device=dev)
    qkv = torch.randn(M, 3 * h, device=dev).to(bf)
    cs3 = torch.zeros(3 * h, device=dev)
    dqa = torch.randn(M, h, device=dev)
    V, Vp = 30522, 30528
    logits = (torch.randn(M, Vp, device=dev) * 3).to(bf)
    labels = torch.randint(0, V, (M,), device=dev)
    lmax, gmax = torch.empty(M, device=dev), torch.empty(M, device=dev)
    packed = torch.empty(M, 2, device=dev)
    K.xent_local(logits, V, labels, 0, lmax, gmax, packed)
    dlog = torch.empty_like(logits)
    cases = {
        "qkv_grad_finish (all 3hb)": (lambda: K.qkv_grad_finish(dqa, qkv, h, cs3), M * h * (4 + 2 + 4)),
        "qkv_grad_finish (q only)": (lambda: K.qkv_grad_finish(dqa, qkv, h, cs3, q_only=True), M * h * 6),
        "xent_local [M,V] bf16": (lambda: K.xent_local(logits, V, labels, 0, lmax, gmax, packed), M * Vp * 2),
        "xent_bwd [M,V] bf16": (lambda: K.xent_bwd(logits, V, labels, 0, gmax, packed, 1.0 / M, dlog), M * Vp * 4),
        "ln_bwd(+resid,dx2,dg,db,ds)": (lambda: K.ln_bwd(dy, x, mean, rstd, gamma, stats, h, res, dx, dx2, dg, db, ds),
                                        M * h * (4 * 4 + 2)),
        "ln_bwd_stats": (lambda: K.ln_bwd_stats(dy, x, mean, rstd, gamma, stats), M * h * 8),
        "ln_fwd(local stats)": (lambda: K.ln_fwd(x, None, h, 1e-5, gamma, beta, y, mean, rstd), M * h * 6),
        "dgelu(in place, colsum)": (lambda: K.dgelu(dact, mid, dact, cs4), M * 4 * h * 6),
        "dgelu(out-of-place)": (lambda: K.dgelu(dact, mid, y.view(-1)[: M * 4 * h // 4].view(M // 4, 4 * h) if False else dact, None), M * 4 * h * 6),
        "colsum bf16 [M,3h]": (lambda: K.colsum(qkv, cs3, accumulate=True), M * 3 * h * 2),
    }
    for name, (fn, nbytes) in cases.items():
        us = bench(fn)
        print(f"{name:32s} {us:8.1f} us  {nbytes / us / 1e3:8.1f} GB/s", flush=True)


if __name__ == "__main__":
    main()
