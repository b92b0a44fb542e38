"""Pin the CPU oracle (oracle/) against golden vectors made by the real reference.

The fixtures in tests/golden/ were produced by oracle/gen_golden.py calling the
unmodified reference package; these tests show the numpy restatement used as
the checker for the CUDA path reproduces them (bookkeeping bit-exact, float64
math to ~1e-12).
"""

import json
import math
from pathlib import Path

import numpy as np
import pytest

import oracle
from oracle import model_ref as M

GOLD = Path(__file__).resolve().parent / "golden"


@pytest.fixture(scope="module")
def book():
    return json.loads((GOLD / "bookkeeping.json").read_text())


@pytest.fixture(scope="module")
def summa():
    return dict(np.load(GOLD / "summa.npz"))


@pytest.fixture(scope="module")
def model():
    return dict(np.load(GOLD / "model.npz")), json.loads((GOLD / "model.json").read_text())


@pytest.fixture(scope="module")
def ops():
    return dict(np.load(GOLD / "layers.npz"))


def test_mesh_groups_and_nodes(book):
    for key, d in book["mesh"].items():
        q = int(key[1:])
        rows, cols = oracle.mesh_groups(q, q)
        assert rows == d["rows"] and cols == d["cols"]
        for ns, nodes in d["natural_nodes"].items():
            assert oracle.node_map(q, q, int(ns), bunched=False) == nodes
        for ns, nodes in d["bunched_nodes"].items():
            if nodes is None:
                with pytest.raises(ValueError):
                    oracle.node_map(q, q, int(ns), bunched=True)
            else:
                assert oracle.node_map(q, q, int(ns), bunched=True) == nodes


def test_scatter_interleave_tokens_vpad(book):
    for key, blocks in book["scatter"].items():
        q = int(key[1:])
        x = np.arange(6 * q * 4 * q, dtype=float).reshape(6 * q, 4 * q)
        mine = [oracle.act_block(x, q, q, f // q, f % q).tolist() for f in range(q * q)]
        assert mine == blocks
    for key, ref in book["interleave"].items():
        h, parts = map(int, key.split("_"))
        w = np.arange(3 * h, dtype=float)
        assert oracle.interleave_qkv(w, parts).tolist() == ref
        assert np.array_equal(oracle.deinterleave_qkv(oracle.interleave_qkv(w, parts), parts), w)
    tok = np.arange(12).reshape(4, 3)
    for key, ref in book["token_block"].items():
        q = int(key[1:])
        assert [oracle.token_block(tok, i, q).tolist() for i in range(q)] == ref
    for key, ref in book["v_padded"].items():
        assert oracle.v_padded(37, int(key[1:])) == ref


def test_summa_products(summa):
    for q in (1, 2, 3):
        a, b, bt, at, dc = (summa[f"q{q}_{k}"] for k in ("a", "b", "bt", "at", "dc"))
        np.testing.assert_allclose(a @ b, summa[f"q{q}_ab"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(a @ bt.T, summa[f"q{q}_abt"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(at.T @ b, summa[f"q{q}_atb"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(dc @ b.T, summa[f"q{q}_ab_da"], rtol=0, atol=1e-12)
        np.testing.assert_allclose(a.T @ dc, summa[f"q{q}_ab_db"], rtol=0, atol=1e-12)


@pytest.mark.parametrize("name", ["small", "wide", "tiny_cfg1", "cli_default"])
def test_model_loss_and_grads(model, name):
    arrays, meta = model
    cfg = M.RefConfig(*meta[name]["dims"])
    params = M.init_params(cfg, meta[name]["seed"])
    for k, s in meta[name]["param_sums"].items():
        assert float(params[k].sum()) == s, k  # PCG64 stream + draw order bit-exact
    tokens, labels = M.sample_data(cfg, meta[name]["seed"])
    assert np.array_equal(tokens, arrays[f"{name}.tokens"]) and np.array_equal(labels, arrays[f"{name}.labels"])
    loss, saved = M.serial_forward(cfg, params, tokens, labels)
    assert abs(loss - meta[name]["loss"]) < 1e-12
    grads = M.serial_backward(cfg, params, saved)
    for k, (s, ss) in meta[name]["grad_sums"].items():
        assert math.isclose(float(grads[k].sum()), s, rel_tol=1e-9, abs_tol=1e-12), k
        assert math.isclose(float((grads[k] ** 2).sum()), ss, rel_tol=1e-9, abs_tol=1e-15), k
    for key, ref in arrays.items():
        if key.startswith(f"{name}.grad."):
            np.testing.assert_allclose(grads[key[len(name) + 6:]], ref, rtol=0, atol=1e-12)
    np.testing.assert_allclose(saved["layers"][0]["y1"], arrays[f"{name}.layer0_y1"], atol=1e-12)
    # mesh runs of the reference agree with its serial model (mesh-size independence)
    for q, ml in meta[name]["mesh_loss"].items():
        assert abs(ml - loss) < 1e-12


def test_operator_fixtures(ops):
    x, dy, gam, bet = ops["ops.x"], ops["ops.dy"], ops["ops.gamma"], ops["ops.beta"]
    cfg = M.RefConfig(b=4, s=4, h=16, n=4, v=14, num_layers=1)
    y, rec = M.layernorm(x, gam, bet, cfg.eps)
    np.testing.assert_allclose(y, ops["ops.ln_y"], atol=1e-12)
    dx, dg, db = M.layernorm_grad(dy, rec)
    np.testing.assert_allclose(dx, ops["ops.ln_dx"], atol=1e-12)
    np.testing.assert_allclose(dg, ops["ops.ln_dg"], atol=1e-12)
    np.testing.assert_allclose(db, ops["ops.ln_db"], atol=1e-12)
    p = M.init_params(cfg, 3)
    pre = "layers.0."
    out, arec = M.attention(x, p[pre + "w_qkv"], p[pre + "b_qkv"], p[pre + "w_dense"], p[pre + "b_dense"], cfg)
    np.testing.assert_allclose(out, ops["ops.attn_out"], atol=1e-12)
    g = M.attention_grad(dy, arec, p[pre + "w_qkv"], p[pre + "w_dense"], cfg)
    for got, key in zip(g, ("attn_dx", "attn_dwqkv", "attn_dbqkv", "attn_dwd", "attn_dbd")):
        np.testing.assert_allclose(got, ops[f"ops.{key}"], atol=1e-12)
    mid = x @ p[pre + "w1"] + p[pre + "b1"]
    act = M.gelu(mid)
    np.testing.assert_allclose(act @ p[pre + "w2"] + p[pre + "b2"], ops["ops.mlp_out"], atol=1e-12)
    dmid = (dy @ p[pre + "w2"].T) * M.gelu_grad(mid)
    np.testing.assert_allclose(dmid @ p[pre + "w1"].T, ops["ops.mlp_dx"], atol=1e-12)
    np.testing.assert_allclose(x.T @ dmid, ops["ops.mlp_dw1"], atol=1e-12)
    np.testing.assert_allclose(act.T @ dy, ops["ops.mlp_dw2"], atol=1e-12)
    for v in (14, 13):
        table = ops[f"ops.v{v}.table"]
        tok, lab = ops[f"ops.v{v}.tokens"], ops[f"ops.v{v}.labels"]
        np.testing.assert_array_equal(table[tok.reshape(-1)], ops[f"ops.v{v}.emb"])
        logits = x @ table.T
        np.testing.assert_allclose(ops[f"ops.v{v}.logits"][:, :v], logits, atol=1e-12)
        losses, sm = M.cross_entropy(logits, lab.reshape(-1))
        assert abs(losses.mean() - float(ops[f"ops.v{v}.ce_loss"])) < 1e-12
        g = sm / losses.size
        g[np.arange(losses.size), lab.reshape(-1)] -= 1.0 / losses.size
        ref = ops[f"ops.v{v}.ce_dlogits"]
        np.testing.assert_allclose(ref[:, :v], g, atol=1e-14)
        assert np.all(ref[:, v:] == 0)
        eg = np.zeros_like(ops[f"ops.v{v}.emb_grad"])
        np.add.at(eg, tok.reshape(-1), dy)
        np.testing.assert_allclose(eg, ops[f"ops.v{v}.emb_grad"], atol=1e-12)


def test_finite_difference_pins_backward():
    cfg = M.RefConfig(b=2, s=4, h=8, n=2, v=11, num_layers=1)
    params = M.init_params(cfg, 4)
    tokens, labels = M.sample_data(cfg, 4)
    loss, saved = M.serial_forward(cfg, params, tokens, labels)
    grads = M.serial_backward(cfg, params, saved)

    def f():
        return M.serial_forward(cfg, params, tokens, labels)[0]

    for key, idx in (("layers.0.w1", (1, 3)), ("layers.0.w_qkv", (2, 17)), ("table", (3, 5)),
                     ("layers.0.ln1_gamma", (4,))):
        fd = M.finite_diff(f, params[key], idx)
        assert abs(fd - grads[key][idx]) < 1e-7 * max(1.0, abs(fd))
