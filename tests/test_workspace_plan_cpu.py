"""Planned workspace capacities (ref model.py:197-222, membuf.py:142-171) on the host.

The kernels are replaced by no-ops (tests/_dryrun.py), so these tests walk the exact
allocation sequence of a training step on a CPU mesh in milliseconds:

* the planned capacity of every capped category equals the measured per-position
  high-water mark (local meshes 1x1 .. 2x4, the SPMD mesh over gloo 1x2 .. 2x4),
  with and without checkpointing and eager SGD;
* planned workspaces enforce the plan: a capacity one scalar short raises
  BufferOverflowError (membuf.py:60-66 of the reference);
* merged forward / backward arenas keep the numbers and lower the peak
  (tests/test_membuf.py:197-213 of the reference).
"""

import json
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from tests._dryrun import no_kernels, peaks

DIMS = [dict(b=4, s=16, h=64, n=8, v=61, num_layers=2), dict(b=4, s=32, h=128, n=4, v=100, num_layers=3),
        dict(b=8, s=16, h=64, n=8, v=1000, num_layers=1)]


def _diff(model, got, ck, eu):
    caps = model.workspace_capacities(ck, eu)
    return {k: (got[k], caps[k]) for k in caps if caps[k] is not None and got[k] != caps[k]}


@pytest.mark.parametrize("rc", [(1, 1), (1, 2), (2, 2), (2, 4)])
@pytest.mark.parametrize("dims", DIMS)
def test_plan_equals_high_water_local(rc, dims):
    if dims["n"] % rc[1] or dims["b"] % rc[0]:
        pytest.skip("mesh does not divide the model")
    for ck in (True, False):
        for eu in (False, True):
            model, got = peaks(dims, rc, ck, eu, planned=True)
            assert not _diff(model, got, ck, eu), (rc, ck, eu, _diff(model, got, ck, eu))


def test_plan_is_enforced():
    import paper_2104_05343_b200 as sg

    dims = DIMS[0]
    with no_kernels():
        mesh = sg.create_mesh(sg.MeshConfig(rows=2, cols=2), device="cpu")
        cfg = sg.ModelConfig(**dims)
        model = sg.MeshModel(mesh, cfg, sg.init_global_params(cfg, 1))
        rng = np.random.default_rng(0)
        tok, lab = rng.integers(0, cfg.v, (cfg.b, cfg.s)), rng.integers(0, cfg.v, (cfg.b, cfg.s))
        for cat in ("forward", "backward", "workspace", "param_grad", "conjunction"):
            caps = model.workspace_capacities(True, False)
            caps[cat] -= 1
            ws = sg.Workspace(mesh.p, capacities=caps, device="cpu")
            with pytest.raises(sg.BufferOverflowError):
                store = sg.CheckpointStore(mesh.p)
                _, saved = model.forward(tok, lab, ws, store=store)
                model.backward(saved, ws)


def test_merged_arenas_same_numbers_smaller_peak():
    ref_model, split = peaks(DIMS[0], (2, 2), True, False)
    _, merged = peaks(DIMS[0], (2, 2), True, False, merge=True)
    assert merged["forward"] < split["forward"] + split["backward"]


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _dist_worker(rank, world, port, rows, cols, out_dir):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2104_05343_b200 as sg

        bad = []
        with no_kernels():
            m = sg.create_mesh(sg.MeshConfig(rows=rows, cols=cols), backend="dist", device="cpu")
            for dims in (DIMS[0], DIMS[2]):
                for ck in (True, False):
                    cfg = sg.ModelConfig(**dims)
                    model = sg.MeshModel(m, cfg, sg.init_global_params(cfg, 1))
                    rng = np.random.default_rng(0)
                    tok, lab = rng.integers(0, cfg.v, (cfg.b, cfg.s)), rng.integers(0, cfg.v, (cfg.b, cfg.s))
                    _, _, ws, _ = sg.run_loss_and_grads(model, tok, lab, checkpointing=ck, planned=True)
                    got = {k: int(v.max()) for k, v in ws.peaks().items()}
                    d = _diff(model, got, ck, False)
                    if d:
                        bad.append([dims["v"], ck, {k: list(v) for k, v in d.items()}])
        (out_dir / f"r{rank}.json").write_text(json.dumps(bad))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols", [(1, 2), (2, 2), (2, 4)])
def test_plan_equals_high_water_dist(tmp_path, rows, cols):
    world = rows * cols
    mp.spawn(_dist_worker, args=(world, _free_port(), rows, cols, tmp_path), nprocs=world, join=True)
    for rank in range(world):
        assert json.loads((tmp_path / f"r{rank}.json").read_text()) == [], rank
