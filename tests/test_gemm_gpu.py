"""tcgen05 GEMM (libsg sg_gemm) against a plain PyTorch fp32 reference.

Covers the three SUMMA operand layouts (AB: K-major A / MN-major B, ABT: both
K-major, ATB: both MN-major), ragged M/N/K, every epilogue and the strided
batched (per-head) form used by the attention kernels.
"""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _k():
    from paper_2104_05343_b200 import kernels

    return kernels


def _rel(x, ref):
    x = x.float()
    ref = ref.float()
    return ((x - ref).abs().max() / ref.abs().max().clamp_min(1e-30)).item()


def _rand(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


@pytest.mark.parametrize("layout", ["ab", "abt", "atb", "atbt"])
@pytest.mark.parametrize("mnk", [(128, 256, 64), (256, 512, 192), (300, 200, 100), (1000, 72, 520),
                                 (64, 1000, 33), (2048, 3072, 1024)])
def test_gemm_layouts(layout, mnk):
    k = _k()
    torch.manual_seed(0)
    M, N, K = mnk
    if layout in ("ab", "abt"):
        a = _rand(M, K)
    else:
        a = _rand(K, M).t()
    if layout in ("ab", "atb"):
        b = _rand(K, N)
    else:
        b = _rand(N, K).t()
    # TMA needs 16-byte aligned leading dims; pad storage where the extent is odd
    out = torch.empty(M, N, device="cuda", dtype=torch.float32)
    try:
        k.gemm(a, b, out)
    except Exception as e:  # unaligned strides are rejected, not silently wrong
        assert "aligned" in str(e)
        return
    ref = a.float() @ b.float()
    assert _rel(out, ref) < 1e-5


def test_gemm_epilogues():
    k = _k()
    torch.manual_seed(1)
    M, N, K = 512, 768, 256
    a, b = _rand(M, K), _rand(K, N)
    bias = torch.randn(N, device="cuda")
    c = torch.randn(M, N, device="cuda")
    ref = a.float() @ b.float()
    out = torch.empty(M, N, device="cuda")
    k.gemm(a, b, out, alpha=0.5, bias=bias, c=c)
    assert _rel(out, 0.5 * ref + bias + c) < 1e-5
    # in-place accumulation (SUMMA step l > 0): C == D
    acc = c.clone()
    k.gemm(a, b, acc, c=acc)
    assert _rel(acc, ref + c) < 1e-5
    # GELU with saved pre-activation, bf16 output
    mid = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    act = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k.gemm(a, b, act, bias=bias, act=k.ACT_GELU, aux=mid)
    x = ref + bias
    assert _rel(mid, x) < 1e-2
    gelu = 0.5 * x * (1 + torch.tanh(math.sqrt(2 / math.pi) * (x + 0.044715 * x ** 3)))
    assert _rel(act, gelu) < 1e-2
    # GELU' epilogue reading the saved pre-activation
    dact = torch.empty(M, N, device="cuda")
    k.gemm(a, b, dact, act=k.ACT_DGELU, aux=mid)
    xm = mid.float()
    t = torch.tanh(math.sqrt(2 / math.pi) * (xm + 0.044715 * xm ** 3))
    dg = 0.5 * (1 + t) + 0.5 * xm * (1 - t * t) * math.sqrt(2 / math.pi) * (1 + 3 * 0.044715 * xm ** 2)
    assert _rel(dact, ref * dg) < 1e-4


def test_gemm_batched_heads():
    """Per-head products on the interleaved QKV block layout (layers.py:404-416)."""
    k = _k()
    torch.manual_seed(2)
    b_loc, n_loc, s, d = 2, 3, 256, 64
    hb = n_loc * d
    qkv = _rand(b_loc * s, 3 * hb)
    q = qkv[:, :hb].view(b_loc, s, n_loc, d).permute(0, 2, 1, 3)       # [b, n, s, d] strided view
    kk = qkv[:, hb:2 * hb].view(b_loc, s, n_loc, d).permute(0, 2, 1, 3)
    v = qkv[:, 2 * hb:].view(b_loc, s, n_loc, d).permute(0, 2, 1, 3)
    scores = torch.empty(b_loc, n_loc, s, s, device="cuda")
    k.gemm(q, kk.transpose(-1, -2), scores, alpha=1 / math.sqrt(d))
    ref = (q.float() @ kk.float().transpose(-1, -2)) / math.sqrt(d)
    assert _rel(scores, ref) < 1e-5
    p = torch.softmax(scores, -1).to(torch.bfloat16)
    ctx = torch.empty(b_loc * s, hb, device="cuda", dtype=torch.bfloat16)
    ctx_v = ctx.view(b_loc, s, n_loc, d).permute(0, 2, 1, 3)
    k.gemm(p, v, ctx_v)
    assert _rel(ctx_v, p.float() @ v.float()) < 1e-2
    # dV = P^T dO: MN-major A (P transposed view), MN-major B
    dv = torch.empty(b_loc, n_loc, s, d, device="cuda")
    k.gemm(p.transpose(-1, -2), ctx_v, dv)
    assert _rel(dv, p.float().transpose(-1, -2) @ ctx_v.float()) < 1e-5


@pytest.mark.parametrize("M,N,K", [(4096, 4096, 4096)])
def test_gemm_large_square(M, N, K):
    k = _k()
    torch.manual_seed(3)
    a, b = _rand(M, K), _rand(K, N)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    k.gemm(a, b, out)
    ref = a.float() @ b.float()
    assert _rel(out, ref) < 1e-2


def test_gemm_colsum_and_bf16_copy():
    k = _k()
    torch.manual_seed(4)
    M, N, K = 700, 520, 256
    a, b = _rand(M, K), _rand(K, N)
    out = torch.empty(M, N, device="cuda")
    out2 = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.zeros(N, device="cuda")
    k.gemm(a, b, out, out2=out2, colsum=cs)
    ref = a.float() @ b.float()
    assert _rel(out, ref) < 1e-5
    assert torch.equal(out2, out.to(torch.bfloat16))
    assert _rel(cs, ref.sum(0)) < 1e-5
    # batched heads, column sums shared over the batch dim (the b_qkv gradient)
    bl, nl, s, d = 2, 3, 128, 64
    x = _rand(bl, nl, s, s)
    y = _rand(bl, nl, s, d)
    o = torch.empty(bl, nl, s, d, device="cuda")
    cs = torch.zeros(1, nl, d, device="cuda")
    k.gemm(x, y, o, colsum=cs)
    assert _rel(cs[0], (x.float() @ y.float()).sum(dim=(0, 2))) < 1e-5


@pytest.mark.parametrize("s", [64, 200, 512])
def test_gemm_softmax_epilogues(s):
    """P = softmax(alpha Q K^T) and dS = P (dP - rowsum(dP P)) alpha, fused in the epilogue."""
    k = _k()
    torch.manual_seed(5)
    bl, nl, d = 2, 4, 64
    alpha = 1 / math.sqrt(d)
    q, kk, do, v = (_rand(bl, nl, s, d) for _ in range(4))
    p = torch.empty(bl, nl, s, s, device="cuda", dtype=torch.bfloat16)
    k.gemm(q, kk.transpose(-1, -2), p, alpha=alpha, mode=k.EPI_SOFTMAX)
    ref = torch.softmax(alpha * (q.float() @ kk.float().transpose(-1, -2)), -1)
    assert (p.float() - ref).abs().max().item() < 4e-3
    ds = torch.empty_like(p)
    dp = do.float() @ v.float().transpose(-1, -2)
    pf = p.float()
    drow = (dp * pf).sum(-1).contiguous()
    k.gemm(do, v.transpose(-1, -2), ds, alpha=alpha, mode=k.EPI_SOFTMAX_BWD, aux=p, rowvec=drow)
    ref_ds = pf * (dp - drow[..., None]) * alpha
    assert _rel(ds, ref_ds) < 1e-2
    # D_i = rowsum(dP P) equals rowsum(dO O) with O = P V (the kernel used by attention backward)
    o = (pf @ v.float()).bfloat16()
    hb = 2 * d
    flat = lambda x: x.permute(0, 2, 1, 3).reshape(bl * s, nl * d).contiguous()  # noqa: E731
    dr = torch.empty(bl, nl, s, device="cuda")
    k.attn_rowdot(flat(do), flat(o), nl, d, s, dr)
    assert _rel(dr, (do.float() * o.float()).sum(-1)) < 1e-4


@pytest.mark.parametrize("M,N,K", [(512, 1024, 4096), (300, 200, 100), (4096, 2048, 8192), (130, 72, 64)])
def test_gemm_layernorm_stats(M, N, K):
    """LayerNorm-backward row statistics accumulated in the dx GEMM's epilogue equal
    the separate stats pass (layers.py:310-351: sum xhat g, sum g with g = dy gamma)."""
    k = _k()
    torch.manual_seed(7)
    a, b = _rand(M, K, scale=0.05), _rand(K, N)
    x = torch.randn(M, N, device="cuda") * 3 + 1
    gamma = torch.randn(N, device="cuda")
    mean = x.mean(1)
    rstd = torch.rsqrt(x.var(1, unbiased=False) + 1e-5)
    dy = torch.empty(M, N, device="cuda")
    stats = torch.zeros(M, 2, device="cuda")
    k.gemm(a, b, dy, ln_stats=(x, gamma, mean, rstd, stats))
    ref = a.float() @ b.float()
    assert _rel(dy, ref) < 4e-5  # fp32 accumulation order over K = 8192
    g = ref * gamma
    xhat = (x - mean[:, None]) * rstd[:, None]
    assert _rel(stats[:, 0], (xhat * g).sum(1)) < 1e-4
    assert _rel(stats[:, 1], g.sum(1)) < 1e-4
    sep = torch.empty(M, 2, device="cuda")
    k.ln_bwd_stats(dy, x, mean, rstd, gamma, sep)
    assert _rel(stats, sep) < 1e-4


@pytest.mark.parametrize("M,N,K", [(700, 520, 256), (4096, 4096, 1024), (1000, 4100, 320)])
def test_gemm_dgelu_colsum_abt(M, N, K):
    """GELU' + column sums on the dX layout (both operands K-major): the 12-warp
    epilogue at pair tiles, ragged edges included, against a PyTorch fp32 reference."""
    k = _k()
    torch.manual_seed(9)
    a, w = _rand(M, K), _rand(N, K)
    mid = _rand(M, N, scale=2.0)
    out = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    cs = torch.zeros(N, device="cuda")
    k.gemm(a, w.t(), out, act=k.ACT_DGELU, aux=mid, colsum=cs)
    xm = mid.float()
    t = torch.tanh(math.sqrt(2 / math.pi) * (xm + 0.044715 * xm ** 3))
    dg = 0.5 * (1 + t) + 0.5 * xm * (1 - t * t) * math.sqrt(2 / math.pi) * (1 + 3 * 0.044715 * xm ** 2)
    ref = (a.float() @ w.float().t()) * dg
    assert _rel(out, ref) < 1e-2
    assert _rel(cs, ref.sum(0)) < 1e-3


@pytest.mark.parametrize("M,N,K", [(1024, 1024, 16384), (1024, 4096, 16384), (300, 260, 4096)])
def test_gemm_in_place_update_with_alpha(M, N, K):
    """w += alpha a^T b in place (the fused SGD step, split-K partials reduce-added with
    alpha applied per split) against w + alpha (a^T b) in fp32."""
    k = _k()
    torch.manual_seed(10)
    a, b = _rand(K, M), _rand(K, N)
    w = torch.randn(M, N, device="cuda")
    want = w + (-0.125) * (a.float().t() @ b.float())
    k.gemm(a.t(), b, w, c=w, alpha=-0.125)
    assert _rel(w, want) < 5e-5  # fp32 accumulation order over K = 16384


_DIE_CASE = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K
torch.manual_seed(2)
M, N, Kd = 16384, 8192, 4096  # 2048 pair tiles: 27.7 waves (a partial last round)
a = torch.randn(M, Kd, device="cuda").bfloat16()
b = torch.randn(Kd, N, device="cuda").bfloat16()
o = torch.empty(M, N, device="cuda", dtype=torch.float32)
K.gemm(a, b, o)
ref = a.float() @ b.float()
err = ((o - ref).abs().max() / ref.abs().max()).item()
torch.cuda.synchronize()
torch.save((o.cpu(), err), sys.argv[1])
'''


@pytest.mark.gpu
def test_gemm_die_local_tile_order(tmp_path):
    """Large pair-tile products run their tiles in die-local streams (SG_GEMM_DIE): the same
    tiles with the same K order, so the result equals the standard order bit for bit."""
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = []
    for die in ("1", "0"):
        f = tmp_path / f"o{die}.pt"
        r = subprocess.run([sys.executable, "-c", _DIE_CASE, str(f)], env=dict(os.environ, SG_GEMM_DIE=die),
                           capture_output=True, text=True, timeout=300, cwd=root)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(torch.load(f))
    assert torch.equal(outs[0][0], outs[1][0])
    assert outs[0][1] < 1e-3, outs[0][1]
