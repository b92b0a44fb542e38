"""Host-only dry run of the model's workspace accounting (test infrastructure).

Every libsg wrapper in ``kernels`` is replaced by a no-op, so a MeshModel on a CPU
local mesh walks exactly the allocation sequence of the GPU path (Workspace.empty /
alloc per category) without computing anything. Used to check the planned
workspace capacities (MeshModel.workspace_capacities) on many shapes quickly.
"""

from __future__ import annotations

import contextlib

import numpy as np


@contextlib.contextmanager
def no_kernels():
    from paper_2104_05343_b200 import kernels as K

    saved = {}
    for name in dir(K):
        fn = getattr(K, name)
        if name.startswith("_") or not callable(fn) or isinstance(fn, type) or name in ("check",):
            continue
        if getattr(fn, "__module__", "") != K.__name__:
            continue
        saved[name] = fn
        setattr(K, name, lambda *a, **k: None)
    try:
        yield
    finally:
        for name, fn in saved.items():
            setattr(K, name, fn)


def peaks(dims: dict, rc=(1, 1), checkpointing=True, eager_update=False, merge=False, planned=False, skip=False):
    import paper_2104_05343_b200 as sg

    with no_kernels():
        mesh = sg.create_mesh(sg.MeshConfig(rows=rc[0], cols=rc[1]), device="cpu")
        cfg = sg.ModelConfig(**dims)
        params = sg.init_global_params(cfg, 1)
        model = sg.MeshModel(mesh, cfg, params, skip_dead_recompute=skip)
        rng = np.random.default_rng(0)
        tok = rng.integers(0, cfg.v, (cfg.b, cfg.s))
        lab = rng.integers(0, cfg.v, (cfg.b, cfg.s))
        _, _, ws, store = sg.run_loss_and_grads(model, tok, lab, checkpointing=checkpointing,
                                                eager_update=eager_update, lr=0.0, merge_fwd_bwd=merge,
                                                planned=planned)
        return model, {k: int(v.max()) for k, v in ws.peaks().items()}
