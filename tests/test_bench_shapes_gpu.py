"""Oracle parity at the benchmarked shapes.

The bench times a BERT-large-shaped stack (h=1024, 16 heads -> head_dim 64, s=512,
v=30522) and the GPT configs use h=4096, 32 heads -> head_dim 128, s=2048. At these
shapes the step runs the flash forward / backward kernels, the fused dQ finish with
the K/V bias column sums (hb % 256 == 0), the LayerNorm-statistics dX epilogue,
split-K weight-gradient products and, in ``train_step``, the SGD update fused into
those products. Every one of them is compared here, end to end, against the float64
oracle (oracle/model_ref.py, a restatement of ref oracle.py:118-205 and
layers.py:380-508) on bf16-rounded parameters:

* loss within 1e-3 relative, every gradient within 2e-2 normwise (north-star BF16
  tolerance), on 1x1 and the simulated 1x2 / 2x2 meshes;
* ``train_step`` (eager SGD, fused into the dW products): (w_after - w_before) / -lr
  equals the oracle gradient to the same tolerance.
"""

import numpy as np
import pytest
import torch

from oracle import model_ref as M
from tests._util import TOL_BF16, bf16_round, mesh, rel

pytestmark = pytest.mark.gpu

BERT = dict(b=2, s=512, h=1024, n=16, v=30522, num_layers=2)
GPT = dict(b=1, s=2048, h=4096, n=32, v=8192, num_layers=1)
_CACHE: dict = {}


def _sg():
    import paper_2104_05343_b200 as sg

    return sg


def _oracle(dims: dict, seed: int):
    key = (tuple(sorted(dims.items())), seed)
    if key not in _CACHE:
        rcfg = M.RefConfig(dims["b"], dims["s"], dims["h"], dims["n"], dims["v"], dims["num_layers"])
        params = {k: bf16_round(v) for k, v in M.init_params(rcfg, seed).items()}
        tokens, labels = M.sample_data(rcfg, seed)
        loss, saved = M.serial_forward(rcfg, params, tokens, labels)
        grads = {k: v for k, v in M.serial_backward(rcfg, params, saved).items() if not k.startswith("_")}
        del saved
        _CACHE[key] = (params, tokens, labels, loss, grads)
    return _CACHE[key]


def _check(got: dict, ref: dict, what: str):
    errs = {k: rel(got[k], ref[k]) for k in ref}
    worst = max(errs, key=errs.get)
    print(f"[parity] {what}: worst gradient {worst} rel {errs[worst]:.3e}")
    bad = {k: v for k, v in errs.items() if v > TOL_BF16}
    assert not bad, (what, bad)
    return max(errs.values())


@pytest.mark.parametrize("rc", [(1, 1), (1, 2), (2, 2)])
@pytest.mark.parametrize("checkpointing", [False, True])
def test_bert_shape_loss_and_grads(rc, checkpointing):
    """h=1024, n=16 (d=64 flash fwd2 / bwd2, qkv_grad_finish + kv_colsum), s=512, v=30522."""
    sg = _sg()
    params, tokens, labels, ref_loss, ref = _oracle(BERT, 31)
    model = sg.MeshModel(mesh(*rc), sg.ModelConfig(**BERT), params)
    loss, grads, _, store = sg.run_loss_and_grads(model, tokens, labels, checkpointing=checkpointing)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3, (loss, ref_loss)
    _check(model.gather_grads(grads), ref, f"bert {rc} ckpt={checkpointing}")
    if checkpointing:
        assert store.count() == 0


@pytest.mark.parametrize("rc", [(1, 1), (2, 2)])
def test_bert_shape_train_step(rc):
    """The bench's step: forward, backward with SGD fused into the weight-gradient
    products (TMA reduce-add into the fp32 masters), table / vector SGD."""
    sg = _sg()
    params, tokens, labels, ref_loss, ref = _oracle(BERT, 31)
    model = sg.MeshModel(mesh(*rc), sg.ModelConfig(**BERT), params)
    lr = 1.0
    ws = model.make_workspace(checkpointing=False)
    loss = float(model.train_step(torch.as_tensor(tokens).cuda(), torch.as_tensor(labels).cuda(), ws, lr).item())
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3
    after = model.gather_params()
    implied = {k: (after[k] - params[k]) / -lr for k in ref}
    _check(implied, ref, f"bert train_step {rc}")


def test_bert_shape_ragged_head_split():
    """hb = h/c not a multiple of 256: the unfused dQ epilogue + column-sum branch."""
    sg = _sg()
    dims = dict(b=2, s=256, h=384, n=6, v=1000, num_layers=1)
    params, tokens, labels, ref_loss, ref = _oracle(dims, 7)
    model = sg.MeshModel(mesh(1, 2), sg.ModelConfig(**dims), params)
    loss, grads, _, _ = sg.run_loss_and_grads(model, tokens, labels, checkpointing=False)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3
    _check(model.gather_grads(grads), ref, "ragged")


@pytest.mark.parametrize("checkpointing", [False, True])
def test_gpt_shape_loss_and_grads(checkpointing):
    """h=4096, n=32 (head_dim 128), s=2048 on 1x1: the GPT configs' attention path."""
    sg = _sg()
    params, tokens, labels, ref_loss, ref = _oracle(GPT, 5)
    model = sg.MeshModel(mesh(1, 1), sg.ModelConfig(**GPT), params)
    loss, grads, _, _ = sg.run_loss_and_grads(model, tokens, labels, checkpointing=checkpointing)
    assert abs(loss - ref_loss) / abs(ref_loss) < 1e-3, (loss, ref_loss)
    _check(model.gather_grads(grads), ref, f"gpt ckpt={checkpointing}")
