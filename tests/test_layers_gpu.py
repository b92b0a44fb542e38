"""2D operators (LayerNorm, attention, MLP, embedding, lm-head + cross entropy)
on r x c meshes vs the float64 oracle; plus the reference-generated q=2 fixtures."""

import math
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import model_ref as M
from tests._util import MESHES, TOL_BF16, bf16_round, mesh, rel

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def _sg():
    import paper_2104_05343_b200 as sg

    return sg


def _vec(sg, vec, m):
    return sg.RowHostedVector.split(vec, m.c, mesh=m)


@pytest.mark.parametrize("rc", MESHES)
def test_layernorm_fwd_bwd(rc):
    sg = _sg()
    from paper_2104_05343_b200 import layers

    r, c = rc
    m = mesh(r, c)
    cfg = sg.ModelConfig(b=4, s=8, h=64, n=8, v=16, num_layers=1)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h)) * 2 + 0.5
    dy = rng.standard_normal(x.shape)
    gam, bet = rng.uniform(0.5, 1.5, cfg.h), rng.standard_normal(cfg.h)
    ws = sg.Workspace(m.p)
    m.stats.clear()
    y, ctx = layers.layernorm_forward(sg.scatter(x, m), _vec(sg, gam, m), _vec(sg, bet, m), cfg, ws,
                                      out_dtype=torch.float32)
    # exactly one packed row all-reduce (layers.py:274-280; tests/test_layers.py:195-204)
    assert m.collective_count("allreduce", "layernorm") == (1 if c > 1 else 0)
    ref, rec = M.layernorm(x, gam, bet, cfg.eps)
    assert rel(sg.gather(y), ref) < 1e-5
    dx, dg, db = layers.layernorm_backward(sg.scatter(dy, m), ctx, cfg, ws)
    rdx, rdg, rdb = M.layernorm_grad(dy, rec)
    assert rel(sg.gather(dx), rdx) < 1e-4
    assert rel(dg.gathered(), rdg) < 1e-4
    assert rel(db.gathered(), rdb) < 1e-5


def test_layernorm_constant_rows_and_golden():
    sg = _sg()
    from paper_2104_05343_b200 import layers

    g = np.load(GOLD / "layers.npz")
    m = mesh(2, 2)
    cfg = sg.ModelConfig(b=4, s=4, h=16, n=4, v=14, num_layers=1)
    ws = sg.Workspace(m.p)
    y, ctx = layers.layernorm_forward(sg.scatter(g["ops.x"], m), _vec(sg, g["ops.gamma"], m),
                                      _vec(sg, g["ops.beta"], m), cfg, ws, out_dtype=torch.float32)
    assert rel(sg.gather(y), g["ops.ln_y"]) < 1e-5
    dx, dg, db = layers.layernorm_backward(sg.scatter(g["ops.dy"], m), ctx, cfg, ws)
    assert rel(sg.gather(dx), g["ops.ln_dx"]) < 1e-4
    assert rel(dg.gathered(), g["ops.ln_dg"]) < 1e-4 and rel(db.gathered(), g["ops.ln_db"]) < 1e-5
    # constant rows normalise to beta (layers tests: constant rows -> 0 with beta 0)
    const = np.tile(np.arange(cfg.b * cfg.s)[:, None].astype(float), (1, cfg.h))
    y, _ = layers.layernorm_forward(sg.scatter(const, m), _vec(sg, np.ones(cfg.h), m), _vec(sg, np.zeros(cfg.h), m),
                                    cfg, ws, out_dtype=torch.float32)
    assert np.max(np.abs(sg.gather(y))) < 1e-2


def _layer_params(sg, m, cfg, seed=3):
    p = M.init_params(M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, 1), seed)
    # randomise the identity vectors too so bias / gamma paths are exercised
    rng = np.random.default_rng(seed)
    for k in ("b_qkv", "b_dense", "b1", "b2", "ln1_beta", "ln2_beta"):
        p["layers.0." + k] = bf16_round(rng.standard_normal(p["layers.0." + k].shape) * 0.1)
    for k in ("w_qkv", "w_dense", "w1", "w2", "table"):
        key = k if k == "table" else "layers.0." + k
        p[key] = bf16_round(p[key])
    return p


@pytest.mark.parametrize("rc", MESHES)
def test_attention_fwd_bwd(rc):
    sg = _sg()
    from paper_2104_05343_b200 import layers

    r, c = rc
    m = mesh(r, c)
    cfg = sg.ModelConfig(b=4, s=32, h=64, n=8, v=16, num_layers=1)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, 1)
    p = _layer_params(sg, m, cfg)
    pre = "layers.0."
    rng = np.random.default_rng(2)
    x = bf16_round(rng.standard_normal((cfg.b * cfg.s, cfg.h)))
    dy = rng.standard_normal(x.shape)
    ws = sg.Workspace(m.p)
    wq = sg.scatter(sg.interleave_qkv(p[pre + "w_qkv"], c), m, layout="weight")
    bq = _vec(sg, sg.interleave_qkv(p[pre + "b_qkv"], c), m)
    wd = sg.scatter(p[pre + "w_dense"], m, layout="weight")
    bd = _vec(sg, p[pre + "b_dense"], m)
    m.stats.clear()
    out, actx = layers.attention_forward(sg.scatter(x, m), wq, bq, wd, bd, cfg, ws)
    assert m.collective_count("allreduce") == 0 and m.collective_count("reduce") == 0
    ref, rec = M.attention(x, p[pre + "w_qkv"], p[pre + "b_qkv"], p[pre + "w_dense"], p[pre + "b_dense"], rcfg)
    assert rel(sg.gather(out), ref) < TOL_BF16
    # saved probabilities are per-head, rows sum to one (tests/test_layers.py:286-303)
    b_loc, n_loc = cfg.b // r, cfg.n // c
    assert tuple(actx.probs[0].shape) == (b_loc, n_loc, cfg.s, cfg.s)
    assert np.allclose(actx.probs[0].float().sum(-1).cpu().numpy(), 1.0, atol=2e-2)
    assert tuple(actx.q_heads[0].shape) == (b_loc, n_loc, cfg.s, cfg.head_dim)
    g = layers.attention_backward(sg.scatter(dy, m), actx, wq, wd, cfg, ws)
    rg = M.attention_grad(dy, rec, p[pre + "w_qkv"], p[pre + "w_dense"], rcfg)
    assert rel(sg.gather(g[0]), rg[0]) < TOL_BF16
    assert rel(sg.deinterleave_qkv(sg.gather(g[1]), c), rg[1]) < TOL_BF16
    assert rel(sg.deinterleave_qkv(g[2].gathered(), c), rg[2]) < TOL_BF16
    assert rel(sg.gather(g[3]), rg[3]) < TOL_BF16
    assert rel(g[4].gathered(), rg[4]) < TOL_BF16


@pytest.mark.parametrize("rc", MESHES)
def test_mlp_fwd_bwd(rc):
    sg = _sg()
    from paper_2104_05343_b200 import layers

    r, c = rc
    m = mesh(r, c)
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=16, num_layers=1)
    p = _layer_params(sg, m, cfg)
    pre = "layers.0."
    rng = np.random.default_rng(4)
    x = bf16_round(rng.standard_normal((cfg.b * cfg.s, cfg.h)))
    dy = rng.standard_normal(x.shape)
    ws = sg.Workspace(m.p)
    w1 = sg.scatter(p[pre + "w1"], m, layout="weight")
    w2 = sg.scatter(p[pre + "w2"], m, layout="weight")
    out, mctx = layers.mlp_forward(sg.scatter(x, m), w1, _vec(sg, p[pre + "b1"], m), w2, _vec(sg, p[pre + "b2"], m),
                                   cfg, ws)
    mid = x @ p[pre + "w1"] + p[pre + "b1"]
    act = M.gelu(mid)
    assert rel(sg.gather(out), act @ p[pre + "w2"] + p[pre + "b2"]) < TOL_BF16
    dxm, gw1, gb1, gw2, gb2 = layers.mlp_backward(sg.scatter(dy, m), mctx, w1, w2, cfg, ws)
    dmid = (dy @ p[pre + "w2"].T) * M.gelu_grad(mid)
    assert rel(sg.gather(dxm), dmid @ p[pre + "w1"].T) < TOL_BF16
    assert rel(sg.gather(gw1), x.T @ dmid) < TOL_BF16
    assert rel(gb1.gathered(), dmid.sum(0)) < TOL_BF16
    assert rel(sg.gather(gw2), act.T @ dy) < TOL_BF16
    assert rel(gb2.gathered(), dy.sum(0)) < 1e-5


@pytest.mark.parametrize("rc", MESHES)
@pytest.mark.parametrize("v", [64, 61])
def test_embedding_lmhead_cross_entropy(rc, v):
    sg = _sg()
    from paper_2104_05343_b200 import layers

    r, c = rc
    m = mesh(r, c)
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=v, num_layers=1)
    rng = np.random.default_rng(5)
    table = bf16_round(rng.uniform(-0.5, 0.5, (v, cfg.h)))
    v_pad = cfg.v_padded(m)
    tpad = np.vstack([table, np.zeros((v_pad - v, cfg.h))])
    T = sg.scatter(tpad, m, layout="weight")
    tok = rng.integers(0, v, (cfg.b, cfg.s))
    tok[0, :3] = 5  # repeated ids accumulate in the backward
    lab = rng.integers(0, v, (cfg.b, cfg.s))
    ws = sg.Workspace(m.p)
    emb = layers.embedding_forward(tok, T, cfg, ws)
    assert np.array_equal(sg.gather(emb), table[tok.reshape(-1)])
    x = bf16_round(rng.standard_normal((cfg.b * cfg.s, cfg.h)))
    logits = layers.lm_head_logits(sg.scatter(x, m), T, ws)
    assert rel(sg.gather(logits)[:, :v], x @ table.T) < 1e-4
    m.stats.clear()
    loss, cctx = layers.cross_entropy_forward(logits, lab, cfg, ws)
    losses, smx = M.cross_entropy(x @ table.T, lab.reshape(-1))
    assert abs(loss - losses.mean()) / abs(losses.mean()) < 1e-5
    dl = layers.cross_entropy_backward(cctx, m, ws, upstream=2.0)
    got = sg.gather(sg.ShardedMatrix(m, cfg.b * cfg.s, v_pad, dl))
    ref = smx * 2.0 / losses.size
    ref[np.arange(losses.size), lab.reshape(-1)] -= 2.0 / losses.size
    assert rel(got[:, :v], ref) < 1e-4
    assert np.all(got[:, v:] == 0)
    dy = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    eg = layers.embedding_backward(sg.scatter(dy, m), tok, T, cfg, ws)
    ref_eg = np.zeros((v_pad, cfg.h))
    np.add.at(ref_eg, tok.reshape(-1), dy)
    assert rel(sg.gather(eg), ref_eg) < 1e-5


def test_errors_on_bad_ids():
    sg = _sg()
    from paper_2104_05343_b200 import layers

    m = mesh(1, 2)
    cfg = sg.ModelConfig(b=2, s=4, h=16, n=2, v=10, num_layers=1)
    T = sg.scatter(np.zeros((10, 16)), m, layout="weight")
    ws = sg.Workspace(m.p)
    with pytest.raises(sg.ConfigError):
        layers.embedding_forward(np.full((2, 4), 10), T, cfg, ws)
    logits = layers.lm_head_logits(sg.scatter(np.zeros((8, 16)), m), T, ws)
    with pytest.raises(sg.ConfigError):
        layers.cross_entropy_forward(logits, np.full((2, 4), -1), cfg, ws)


def test_uniform_and_dominant_logits():
    """Uniform logits -> ln v; one dominant logit -> ~0 loss (tests/test_layers.py:523-540)."""
    sg = _sg()
    from paper_2104_05343_b200 import layers

    m = mesh(1, 2)
    cfg = sg.ModelConfig(b=2, s=4, h=16, n=2, v=2, num_layers=1)
    ws = sg.Workspace(m.p)
    lab = np.zeros((2, 4), dtype=np.int64)
    lg = sg.scatter(np.zeros((8, 2)), m)
    loss, _ = layers.cross_entropy_forward(lg, lab, cfg, ws)
    assert abs(loss - math.log(2)) < 1e-6
    big = np.zeros((8, 2))
    big[:, 0] = 40.0
    loss, _ = layers.cross_entropy_forward(sg.scatter(big, m), lab, cfg, ws)
    assert loss < 1e-9 + 1e-6


def test_golden_operator_fixtures_q2():
    """Per-operator outputs of the reference mesh at q=2 (oracle/gen_golden.py)."""
    sg = _sg()
    from paper_2104_05343_b200 import layers

    g = np.load(GOLD / "layers.npz")
    m = mesh(2, 2)
    cfg = sg.ModelConfig(b=4, s=4, h=16, n=4, v=14, num_layers=1)  # head_dim 4: CUDA-core GEMM path
    params = sg.init_global_params(cfg, 3)
    model = sg.MeshModel(m, cfg, params)
    lp = model.layers[0].params
    ws = sg.Workspace(m.p)
    x = sg.scatter(g["ops.x"], m)
    out, actx = layers.attention_forward(x, lp.w_qkv, lp.b_qkv, lp.w_dense, lp.b_dense, cfg, ws)
    assert rel(sg.gather(out), g["ops.attn_out"]) < TOL_BF16
    gr = layers.attention_backward(sg.scatter(g["ops.dy"], m), actx, lp.w_qkv, lp.w_dense, cfg, ws)
    assert rel(sg.gather(gr[0]), g["ops.attn_dx"]) < TOL_BF16
    assert rel(sg.deinterleave_qkv(sg.gather(gr[1]), 2), g["ops.attn_dwqkv"]) < TOL_BF16
    out, mctx = layers.mlp_forward(sg.scatter(g["ops.x"], m), lp.w1, lp.b1, lp.w2, lp.b2, cfg, ws)
    assert rel(sg.gather(out), g["ops.mlp_out"]) < TOL_BF16
    dxm, gw1, gb1, gw2, gb2 = layers.mlp_backward(sg.scatter(g["ops.dy"], m), mctx, lp.w1, lp.w2, cfg, ws)
    assert rel(sg.gather(dxm), g["ops.mlp_dx"]) < TOL_BF16
    assert rel(sg.gather(gw1), g["ops.mlp_dw1"]) < TOL_BF16
    assert rel(sg.gather(gw2), g["ops.mlp_dw2"]) < TOL_BF16
    for v in (14, 13):
        cfgv = sg.ModelConfig(b=4, s=4, h=16, n=4, v=v, num_layers=1)
        mv = sg.MeshModel(m, cfgv, sg.init_global_params(cfgv, 7))
        emb = layers.embedding_forward(g[f"ops.v{v}.tokens"], mv.table, cfgv, ws)
        assert rel(sg.gather(emb), g[f"ops.v{v}.emb"]) < 1e-6
        logits = layers.lm_head_logits(sg.scatter(g["ops.x"], m), mv.table, ws)
        assert rel(sg.gather(logits), g[f"ops.v{v}.logits"]) < TOL_BF16
        loss, cctx = layers.cross_entropy_forward(logits, g[f"ops.v{v}.labels"], cfgv, ws)
        assert abs(loss - float(g[f"ops.v{v}.ce_loss"])) / float(g[f"ops.v{v}.ce_loss"]) < TOL_BF16
        dl = layers.cross_entropy_backward(cctx, m, ws)
        got = sg.gather(sg.ShardedMatrix(m, 16, cfgv.v_padded(m), dl))
        assert rel(got, g[f"ops.v{v}.ce_dlogits"]) < TOL_BF16
        eg = layers.embedding_backward(sg.scatter(g["ops.dy"], m), g[f"ops.v{v}.tokens"], mv.table, cfgv, ws)
        assert rel(sg.gather(eg), g[f"ops.v{v}.emb_grad"]) < 1e-5


_DET_EMBED = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K
torch.manual_seed(5)
n, v, hc = 3000, 97, 320
ids = torch.randint(0, v, (n,), device="cuda")
ids[:400] = 7  # a hot row: more matches than one flush list
dout = torch.randn(n, hc, device="cuda")
ref = torch.zeros(v, hc, dtype=torch.float64, device="cuda").index_add_(0, ids, dout.double())
outs = []
for _ in range(2):
    g = torch.zeros(v, hc, device="cuda")
    K.embed_bwd(ids, 0, v, dout, g)
    outs.append(g)
torch.cuda.synchronize()
err = ((outs[0].double() - ref).abs().max() / ref.abs().max()).item()
same = bool(torch.equal(outs[0], outs[1]))
print(f"{err:.3e} {same}")
'''


@pytest.mark.gpu
def test_embedding_backward_deterministic():
    """SG_DETERMINISTIC=1: the embedding backward sums each row in token order (bit-identical
    across calls) and matches the float64 index-add."""
    import os
    import subprocess
    import sys

    env = dict(os.environ, SG_DETERMINISTIC="1")
    out = subprocess.run([sys.executable, "-c", _DET_EMBED], env=env, capture_output=True, text=True, timeout=300,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert out.returncode == 0, out.stderr[-2000:]
    err, same = out.stdout.split()
    assert float(err) < 1e-5 and same == "True", out.stdout
