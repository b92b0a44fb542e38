"""End-to-end loss and every gradient of the 2D model vs the float64 oracle
(and the reference-generated golden model fixtures), on 1x1, 1x2, 2x2, 2x4."""

import json
from pathlib import Path

import numpy as np
import pytest

from oracle import model_ref as M
from tests._util import MESHES, TOL_BF16, bf16_round, mesh, rel

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).parent / "golden"


def _sg():
    import paper_2104_05343_b200 as sg

    return sg


def _compare_grads(sg, grads, ref, tol=TOL_BF16):
    worst = {}
    for k, g in grads.items():
        worst[k] = rel(g, ref[k])
    bad = {k: v for k, v in worst.items() if v > tol}
    assert not bad, bad


@pytest.mark.parametrize("rc", MESHES)
@pytest.mark.parametrize("checkpointing", [True, False])
def test_model_vs_oracle(rc, checkpointing):
    sg = _sg()
    r, c = rc
    m = mesh(r, c)
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=61, num_layers=2)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers)
    params = {k: bf16_round(v) for k, v in M.init_params(rcfg, 23).items()}
    tokens, labels = M.sample_data(rcfg, 23)
    model = sg.MeshModel(m, cfg, params)
    loss, grads, ws, store = sg.run_loss_and_grads(model, tokens, labels, checkpointing=checkpointing)
    ref_loss, saved = M.serial_forward(rcfg, params, tokens, labels)
    ref = M.serial_backward(rcfg, params, saved)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3
    _compare_grads(sg, model.gather_grads(grads), {k: v for k, v in ref.items() if not k.startswith("_")})
    if checkpointing:
        assert store.count() == 0  # every checkpoint consumed by the recompute


@pytest.mark.parametrize("name", ["wide", "cli_default", "tiny_cfg1", "small"])
def test_golden_model(name):
    """Reference-generated loss / gradients (q = 1 and 2 meshes of the reference)."""
    sg = _sg()
    arrays = np.load(GOLD / "model.npz")
    meta = json.loads((GOLD / "model.json").read_text())[name]
    b, s, h, n, v, L = meta["dims"]
    cfg = sg.ModelConfig(b=b, s=s, h=h, n=n, v=v, num_layers=L)
    params = sg.init_global_params(cfg, meta["seed"])
    for k, ps in meta["param_sums"].items():
        assert float(params[k].sum()) == ps  # bit-exact init stream
    tokens, labels = arrays[f"{name}.tokens"], arrays[f"{name}.labels"]
    for rc in ((1, 1), (2, 2)):
        m = mesh(*rc)
        if b % rc[0] or n % rc[1] or (h // rc[1]) % (h // n):
            continue
        model = sg.MeshModel(m, cfg, params)
        loss, grads, _, _ = sg.run_loss_and_grads(model, tokens, labels)
        assert abs(loss - meta["loss"]) / meta["loss"] < TOL_BF16
        g = model.gather_grads(grads)
        for k, (gs, gss) in meta["grad_sums"].items():
            # sum of squares is a norm check that does not cancel
            assert abs(float((g[k] ** 2).sum()) - gss) / max(gss, 1e-30) < 4 * TOL_BF16, k
        for key in arrays.files:
            if key.startswith(f"{name}.grad."):
                k = key[len(name) + 6:]
                assert rel(g[k], arrays[key]) < TOL_BF16, (rc, k)


def test_mesh_size_independent_loss():
    """The loss does not depend on the mesh shape (tests/test_model.py:67-75)."""
    sg = _sg()
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=40, num_layers=1)
    params = sg.init_global_params(cfg, 5)
    rng = np.random.default_rng(6)
    tok, lab = rng.integers(0, 40, (4, 16)), rng.integers(0, 40, (4, 16))
    losses = []
    for rc in MESHES:
        model = sg.MeshModel(mesh(*rc), cfg, params)
        losses.append(sg.run_loss_and_grads(model, tok, lab)[0])
    assert max(losses) - min(losses) < 1e-3 * abs(losses[0])


def test_zero_weights_loss_is_log_v():
    """Zero weights and table give uniform logits: loss = ln v (tests/test_oracle.py:34-41)."""
    sg = _sg()
    cfg = sg.ModelConfig(b=2, s=8, h=32, n=4, v=24, num_layers=1)
    params = {k: np.zeros_like(v) if k.startswith("layers") and "gamma" not in k else v
              for k, v in sg.init_global_params(cfg, 1).items()}
    params["table"] = np.zeros_like(params["table"])
    model = sg.MeshModel(mesh(1, 2), cfg, params)
    tok = np.zeros((2, 8), dtype=np.int64)
    loss, _, _, _ = sg.run_loss_and_grads(model, tok, tok)
    assert abs(loss - np.log(24)) < 1e-5


def test_sgd_step_reduces_loss_and_train_step():
    sg = _sg()
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=32, num_layers=2)
    params = sg.init_global_params(cfg, 9)
    rng = np.random.default_rng(1)
    tok, lab = rng.integers(0, 32, (4, 16)), rng.integers(0, 32, (4, 16))
    model = sg.MeshModel(mesh(2, 2), cfg, params)
    l0, grads, _, _ = sg.run_loss_and_grads(model, tok, lab)
    model.apply_sgd(grads, 0.5)
    ws = model.make_workspace()
    l1 = float(model.train_step(tok, lab, ws, lr=0.5).item())
    l2 = float(model.train_step(tok, lab, ws, lr=0.5).item())
    assert l1 < l0 and l2 < l1
    # the fused-update step equals reference-order update followed by forward
    ref = sg.MeshModel(mesh(2, 2), cfg, params)
    _, g, _, _ = sg.run_loss_and_grads(ref, tok, lab)
    ref.apply_sgd(g, 0.5)
    p_ref = ref.gather_params()
    model2 = sg.MeshModel(mesh(2, 2), cfg, params)
    model2.train_step(tok, lab, model2.make_workspace(), lr=0.5)
    p_got = model2.gather_params()
    for k in p_ref:
        assert rel(p_got[k], p_ref[k]) < 1e-5, k


@pytest.mark.parametrize("rc", [(1, 1), (2, 2)])
@pytest.mark.parametrize("d", [64, 128])
def test_infer_matches_oracle_loss(rc, d):
    """Forward-only inference (MeshModel.infer, no saved state) gives the oracle loss;
    head_dim 128 runs the d=128 flash forward (model.py:296-324)."""
    import torch

    sg = _sg()
    m = mesh(*rc)
    n = 2 * rc[1]
    h = n * d
    cfg = sg.ModelConfig(b=4, s=128, h=h, n=n, v=64, num_layers=1)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers)
    params = {k: bf16_round(v) for k, v in M.init_params(rcfg, 5).items()}
    tokens, labels = M.sample_data(rcfg, 5)
    model = sg.MeshModel(m, cfg, params)
    ws = model.make_workspace()
    loss = float(model.infer(torch.as_tensor(tokens), torch.as_tensor(labels), ws).item())
    ref_loss, _ = M.serial_forward(rcfg, params, tokens, labels)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3


def test_head_dim_128_training_vs_oracle():
    """d = 128: flash forward, backward through the rebuilt probabilities."""
    sg = _sg()
    m = mesh(1, 2)
    cfg = sg.ModelConfig(b=2, s=128, h=512, n=4, v=64, num_layers=1)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers)
    params = {k: bf16_round(v) for k, v in M.init_params(rcfg, 9).items()}
    tokens, labels = M.sample_data(rcfg, 9)
    model = sg.MeshModel(m, cfg, params)
    loss, grads, _, _ = sg.run_loss_and_grads(model, tokens, labels, checkpointing=False)
    ref_loss, saved = M.serial_forward(rcfg, params, tokens, labels)
    ref = M.serial_backward(rcfg, params, saved)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3
    _compare_grads(sg, model.gather_grads(grads), {k: v for k, v in ref.items() if not k.startswith("_")})


def test_checkpoint_file_across_meshes(tmp_path):
    """A model saved from a 2x2 mesh and reloaded on 1x2 keeps its parameters and loss."""
    import torch

    sg = _sg()
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=61, num_layers=2)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers)
    params = {k: bf16_round(v) for k, v in M.init_params(rcfg, 4).items()}
    tokens, labels = M.sample_data(rcfg, 4)
    a = sg.MeshModel(mesh(2, 2), cfg, params)
    path = tmp_path / "m.bin"
    a.save(path)
    b = sg.MeshModel.load(path, mesh(1, 2))
    pa, pb = a.gather_params(), b.gather_params()
    for k in pa:
        np.testing.assert_array_equal(pa[k], pb[k])
    la = float(a.infer(torch.as_tensor(tokens), torch.as_tensor(labels), a.make_workspace()).item())
    lb = float(b.infer(torch.as_tensor(tokens), torch.as_tensor(labels), b.make_workspace()).item())
    assert abs(la - lb) / abs(la) < 1e-3


@pytest.mark.parametrize("rc", [(1, 1), (1, 2), (2, 2), (2, 4)])
@pytest.mark.parametrize("checkpointing", [False, True])
def test_classifier_branch_vs_reference(rc, checkpointing):
    """Position-0 binary classifier head (model.py:238-292): loss and every gradient,
    cls_w included, against the reference's own q = 2 run (tests/golden/model_cls.npz)."""
    sg = _sg()
    g = np.load(GOLD / "model_cls.npz")
    cfg = sg.ModelConfig(b=4, s=8, h=32, n=4, v=24, num_layers=1)
    params = {k[len("param."):]: g[k] for k in g.files if k.startswith("param.")}
    model = sg.MeshModel(mesh(*rc), cfg, params, classifier=True)
    loss, grads, _, _ = sg.run_loss_and_grads(model, g["tokens"], g["labels"], checkpointing=checkpointing,
                                              cls_labels=g["cls_labels"])
    assert abs(loss - float(g["loss"])) / abs(float(g["loss"])) < 1e-2
    got = model.gather_grads(grads)
    assert set(got) == {k[len("grad."):] for k in g.files if k.startswith("grad.")}
    _compare_grads(sg, got, {k[len("grad."):]: g[k] for k in g.files if k.startswith("grad.")})
    with pytest.raises(sg.ConfigError):
        model.forward(g["tokens"], g["labels"], model.make_workspace())  # cls_labels missing


def test_out_of_range_device_ids_raise():
    """Token ids / labels outside [0, v) raise ConfigError (layers.py:164-165, 552-553)
    also for device tensors: the operator API checks on the device and reads the flag
    back; the model defers the read to the loss read-back / check_inputs()."""
    import torch

    sg = _sg()
    from paper_2104_05343_b200 import layers

    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=40, num_layers=1)
    params = sg.init_global_params(cfg, 3)
    model = sg.MeshModel(mesh(1, 2), cfg, params)
    rng = np.random.default_rng(2)
    tok = torch.as_tensor(rng.integers(0, 40, (4, 16))).cuda()
    lab = torch.as_tensor(rng.integers(0, 40, (4, 16))).cuda()
    ws = model.make_workspace()
    model.forward(tok, lab, ws)  # in range: no error
    model.check_inputs()
    bad_tok, bad_lab = tok.clone(), lab.clone()
    bad_tok[1, 3] = 40
    bad_lab[2, 5] = -1
    with pytest.raises(sg.ConfigError):
        model.forward(bad_tok, lab, model.make_workspace())
    with pytest.raises(sg.ConfigError):
        model.forward(tok, bad_lab, model.make_workspace())
    model.train_step(bad_tok, lab, model.make_workspace(), lr=0.1)
    with pytest.raises(sg.ConfigError):
        model.check_inputs()
    model.check_inputs()  # the flag was cleared
    with pytest.raises(sg.ConfigError):
        layers.embedding_forward(bad_tok, model.table, cfg, ws)
