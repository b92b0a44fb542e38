"""Flash-style attention kernels vs a plain PyTorch fp32 reference."""

import math

import pytest
import torch

pytestmark = pytest.mark.gpu


def _ref(qkv, b, s, nh, d):
    hb = nh * d
    q, k, v = (qkv[:, i * hb:(i + 1) * hb].float().view(b, s, nh, d).permute(0, 2, 1, 3) for i in range(3))
    sc = (q @ k.transpose(-1, -2)) / math.sqrt(d)
    p = torch.softmax(sc, -1)
    o = (p @ v).permute(0, 2, 1, 3).reshape(b * s, hb)
    lse = torch.logsumexp(sc, -1)
    return o, lse, p


@pytest.mark.parametrize("b,s,nh,d", [(2, 512, 4, 64), (3, 200, 2, 64), (1, 384, 2, 128), (2, 1024, 2, 64),
                                      (1, 2048, 2, 128), (2, 64, 3, 64)])
def test_flash_forward(b, s, nh, d):
    from paper_2104_05343_b200 import kernels as K

    torch.manual_seed(0)
    hb = nh * d
    qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
    out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, nh, s, device="cuda")
    K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
    o, l, _ = _ref(qkv, b, s, nh, d)
    assert (out.float() - o).abs().max().item() / o.abs().max().item() < 1e-2
    assert (lse - l).abs().max().item() < 1e-2


@pytest.mark.parametrize("b,s,nh,d", [(2, 512, 4, 64), (3, 200, 2, 64), (2, 1024, 2, 64), (2, 64, 3, 64),
                                      (1, 130, 1, 64), (1, 2048, 2, 64), (40, 128, 8, 64),
                                      (1, 2048, 2, 128), (2, 512, 2, 128), (3, 200, 2, 128), (1, 130, 1, 128),
                                      (40, 128, 4, 128), (1, 384, 4, 128)])
def test_flash_backward(b, s, nh, d):
    from paper_2104_05343_b200 import kernels as K

    torch.manual_seed(1)
    hb = nh * d
    qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
    dout = torch.randn(b * s, hb, device="cuda").bfloat16()
    out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, nh, s, device="cuda")
    K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
    drow = torch.empty(b, nh, s, device="cuda")
    K.attn_rowdot(dout, out, nh, d, s, drow)
    dq = torch.zeros(b * s, hb, device="cuda")
    dqkv = torch.full((b * s, 3 * hb), float("nan"), device="cuda", dtype=torch.bfloat16)
    kv_cs = torch.zeros(2 * hb, device="cuda")
    K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv, kv_colsum=kv_cs)
    torch.cuda.synchronize()
    # fused K / V bias-gradient column sums equal the sums of the bf16 dK, dV written
    want_cs = dqkv[:, hb:].float().sum(0)
    assert (kv_cs - want_cs).abs().max().item() <= 1e-3 * want_cs.abs().max().item() + 1e-4
    # the dQ finishing pass: bf16 dQ and its column sums only
    q_cs = torch.zeros(3 * hb, device="cuda")
    dqkv2 = dqkv.clone()
    if hb % 256 == 0:
        K.qkv_grad_finish(dq, dqkv2, hb, q_cs, q_only=True)
        assert torch.equal(dqkv2[:, :hb], dq.to(torch.bfloat16))
        assert torch.equal(dqkv2[:, hb:], dqkv[:, hb:])
        # (the dQ part is summed from the fp32 accumulator, before the bf16 rounding)
        assert (q_cs[:hb] - dq.sum(0)).abs().max().item() <= 1e-4 * q_cs.abs().max().item() + 1e-5
        assert q_cs[hb:].abs().max().item() == 0.0

    x = qkv.float().requires_grad_(True)
    o, _, _ = _ref(x, b, s, nh, d)
    o.backward(dout.float())
    g = x.grad
    for i, got in enumerate((dq, dqkv[:, hb:2 * hb].float(), dqkv[:, 2 * hb:].float())):
        want = g[:, i * hb:(i + 1) * hb]
        err = (got - want).abs().max().item() / want.abs().max().item()
        assert err < 2e-2, (i, err)


@pytest.mark.parametrize("d", [64, 128])
def test_flash_backward_batch_chunks(d, monkeypatch):
    """Large batches run as several launches over batch chunks (bounded per-CTA item
    tables); forcing tiny chunks gives the same gradients as one launch."""
    from paper_2104_05343_b200 import kernels as K

    torch.manual_seed(3)
    b, s, nh = 9, 256, 2
    hb = nh * d
    qkv = torch.randn(b * s, 3 * hb, device="cuda").bfloat16()
    dout = torch.randn(b * s, hb, device="cuda").bfloat16()
    out = torch.empty(b * s, hb, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(b, nh, s, device="cuda")
    K.flash_attn_fwd(qkv, b, s, nh, d, out, lse)
    drow = torch.empty(b, nh, s, device="cuda")
    K.attn_rowdot(dout, out, nh, d, s, drow)
    res = []
    for items_max in (None, str(2 * nh * 2)):  # two sequences per launch
        if items_max:
            monkeypatch.setenv("SG_FLASH_ITEMS_MAX", items_max)
        dq = torch.zeros(b * s, hb, device="cuda")
        dqkv = torch.zeros(b * s, 3 * hb, device="cuda", dtype=torch.bfloat16)
        cs = torch.zeros(2 * hb, device="cuda")
        K.flash_attn_bwd(qkv, dout, lse, drow, b, s, nh, d, dq, dqkv, kv_colsum=cs)
        torch.cuda.synchronize()
        res.append((dq, dqkv[:, hb:].float(), cs))
    monkeypatch.delenv("SG_FLASH_ITEMS_MAX", raising=False)
    for a, c in zip(res[0], res[1]):
        assert (a - c).abs().max().item() <= 1e-5 * a.abs().max().item() + 1e-6
