"""Memory-plan features on the GPU path, against the reference's own properties
(tests/test_membuf.py:176-240 of the reference): skip_dead_recompute drops the 4h->h
product from the recompute without changing any gradient; merged forward / backward
arenas change no number; eager SGD on the checkpointed path updates the weights and
keeps one layer of parameter gradients; planned capacities hold on the real step."""

import numpy as np
import pytest

from oracle import model_ref as M
from tests._util import bf16_round, mesh, rel

pytestmark = pytest.mark.gpu


def _sg():
    import paper_2104_05343_b200 as sg

    return sg


def _setup(rc=(2, 2), seed=3):
    sg = _sg()
    cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=61, num_layers=2)
    rcfg = M.RefConfig(cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers)
    params = {k: bf16_round(v) for k, v in M.init_params(rcfg, seed).items()}
    tokens, labels = M.sample_data(rcfg, seed)
    return sg, cfg, params, tokens, labels


def test_skip_dead_recompute_same_grads_fewer_macs():
    sg, cfg, params, tokens, labels = _setup()
    ref = sg.MeshModel(mesh(2, 2), cfg, params)
    l1, g1, _, _ = sg.run_loss_and_grads(ref, tokens, labels, checkpointing=True)
    m_skip = mesh(2, 2)
    skip = sg.MeshModel(m_skip, cfg, params, skip_dead_recompute=True)
    l2, g2, _, _ = sg.run_loss_and_grads(skip, tokens, labels, checkpointing=True)
    assert abs(l1 - l2) <= 1e-6 * abs(l1)
    ga, gb = ref.gather_grads(g1), skip.gather_grads(g2)
    for k in ga:
        assert rel(gb[k], ga[k]) < 1e-5, k
    # the 4h->h product (4 b s h^2 / p MACs per layer) is skipped in each recompute
    saved = cfg.num_layers * 4 * cfg.b * cfg.s * cfg.h * cfg.h // 4
    assert np.all(ref.mesh.ledger.macs - m_skip.ledger.macs == saved)


def test_merged_arenas_same_numbers():
    sg, cfg, params, tokens, labels = _setup(seed=7)
    a = sg.MeshModel(mesh(2, 2), cfg, params)
    la, ga, ws_a, _ = sg.run_loss_and_grads(a, tokens, labels, merge_fwd_bwd=True)
    b = sg.MeshModel(mesh(2, 2), cfg, params)
    lb, gb, ws_b, _ = sg.run_loss_and_grads(b, tokens, labels)
    assert abs(la - lb) <= 1e-6 * abs(lb)
    x, y = a.gather_grads(ga), b.gather_grads(gb)
    for k in y:
        assert rel(x[k], y[k]) < 1e-5, k
    assert int(ws_a.peak("forward").max()) < int(ws_b.peak("forward").max()) + int(ws_b.peak("backward").max())


def test_eager_update_checkpointed_applies_sgd():
    sg, cfg, params, tokens, labels = _setup(seed=6)
    model = sg.MeshModel(mesh(2, 2), cfg, params)
    before = model.gather_params()
    _, grads, ws, _ = sg.run_loss_and_grads(model, tokens, labels, eager_update=True, lr=0.5)
    after = model.gather_params()
    assert all(g is None for g in grads.layers)
    ref = sg.MeshModel(mesh(2, 2), cfg, params)
    _, g, _, _ = sg.run_loss_and_grads(ref, tokens, labels)
    gg = ref.gather_grads(g)
    for k in gg:
        if k.startswith("layers."):
            assert rel((after[k] - before[k]) / -0.5, gg[k]) < 2e-2, k
    # one layer's vector gradients (+ the lm-head's b2 column sums) at a time, no weight gradients
    assert int(ws.peak("param_grad").max()) == model.workspace_capacities(True, True)["param_grad"]


@pytest.mark.parametrize("rc", [(1, 1), (1, 2), (2, 2), (2, 4)])
def test_planned_capacities_hold(rc):
    sg, cfg, params, tokens, labels = _setup(rc)
    model = sg.MeshModel(mesh(*rc), cfg, params)
    for ck in (True, False):
        _, _, ws, _ = sg.run_loss_and_grads(model, tokens, labels, checkpointing=ck, planned=True)
        caps = model.workspace_capacities(ck)
        for cat, cap in caps.items():
            if cap is not None:
                assert int(ws.peak(cat).max()) == cap, (cat, rc, ck)
