"""The SPMD ("dist") mesh backend: one process per mesh position.

* CPU: gloo process groups with world sizes 2 / 4 / 8 check the row / column
  communicators, broadcast roots and all-reduce folds of the runtime.
* GPU: 4 processes (2x2 mesh) share one B200 through gloo with CUDA tensors
  and run the SUMMA forms and a full training step; results must equal the
  oracle like the single-controller path (NCCL needs one GPU per rank, which
  the round's single-GPU box does not have).
"""

import json
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _init(rank, world, port):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)


def _collectives_worker(rank, world, port, rows, cols, out_dir):
    import paper_2104_05343_b200 as sg

    _init(rank, world, port)
    try:
        m = sg.create_mesh(sg.MeshConfig(rows=rows, cols=cols), backend="dist", device="cpu")
        f = m.my_flat
        i, j = divmod(f, cols)
        src = [None] * m.p
        src[f] = torch.full((3, 5), float(f))
        res = {}
        got = m.bcast_row(cols - 1, src, (3, 5), torch.float32)
        res["bcast_row"] = float(got[f][0, 0])
        got = m.bcast_col(0, src, (3, 5), torch.float32)
        res["bcast_col"] = float(got[f][0, 0])
        bufs = [None] * m.p
        bufs[f] = torch.full((4,), float(f + 1))
        m.allreduce_row(bufs)
        res["ar_row"] = float(bufs[f][0])
        bufs[f] = torch.full((4,), float(f + 1))
        m.allreduce_col(bufs, op="max")
        res["ar_col_max"] = float(bufs[f][0])
        res["flat"] = f
        (out_dir / f"r{rank}.json").write_text(json.dumps(res))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("rows,cols", [(1, 2), (2, 2), (2, 4)])
def test_gloo_collectives_cpu(tmp_path, rows, cols):
    world = rows * cols
    mp.spawn(_collectives_worker, args=(world, _free_port(), rows, cols, tmp_path), nprocs=world, join=True)
    for rank in range(world):
        res = json.loads((tmp_path / f"r{rank}.json").read_text())
        f = res["flat"]
        i, j = divmod(f, cols)
        assert res["bcast_row"] == i * cols + cols - 1
        assert res["bcast_col"] == j
        assert res["ar_row"] == sum(i * cols + jj + 1 for jj in range(cols))
        assert res["ar_col_max"] == (rows - 1) * cols + j + 1


def _gpu_worker(rank, world, port, rows, cols, out_dir):
    import paper_2104_05343_b200 as sg
    from oracle import model_ref as M

    _init(rank, world, port)
    try:
        torch.cuda.set_device(0)
        m = sg.create_mesh(sg.MeshConfig(rows=rows, cols=cols), backend="dist")
        rng = np.random.default_rng(0)
        bf = lambda a: torch.as_tensor(a, dtype=torch.float32).bfloat16().double().numpy()  # noqa: E731
        a = bf(rng.standard_normal((16 * rows, 16 * cols)))
        b = bf(rng.standard_normal((16 * cols, 24 * cols)))
        bt = bf(rng.standard_normal((24 * cols, 16 * cols)))
        ws = sg.Workspace(m.p)
        A, B, BT = sg.scatter(a, m), sg.scatter(b, m, layout="weight"), sg.scatter(bt, m, layout="weight")
        err = {}

        def rel(x, r):
            return float(np.max(np.abs(x - r)) / np.max(np.abs(r)))

        err["ab"] = rel(sg.gather(sg.summa_ab(A, B, ws)), a @ b)
        err["abt"] = rel(sg.gather(sg.summa_abt(A, BT, ws)), a @ bt.T)
        a2 = bf(rng.standard_normal((16 * rows, 24 * cols)))
        err["atb"] = rel(sg.gather(sg.summa_atb(A, sg.scatter(a2, m), ws)), a.T @ a2)
        cfg = sg.ModelConfig(b=4, s=16, h=64, n=8, v=61, num_layers=2)
        rcfg = M.RefConfig(4, 16, 64, 8, 61, 2)
        params = {k: bf(v) for k, v in M.init_params(rcfg, 23).items()}
        tokens, labels = M.sample_data(rcfg, 23)
        model = sg.MeshModel(m, cfg, params)
        loss, grads, _, _ = sg.run_loss_and_grads(model, tokens, labels, checkpointing=True)
        ref_loss, saved = M.serial_forward(rcfg, params, tokens, labels)
        ref = M.serial_backward(rcfg, params, saved)
        err["loss"] = abs(loss - ref_loss) / abs(ref_loss)
        g = model.gather_grads(grads)
        err["grads"] = max(rel(g[k], ref[k]) for k in g)
        (out_dir / f"r{rank}.json").write_text(json.dumps(err))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("rows,cols", [(1, 2), (2, 2)])
def test_dist_backend_on_one_gpu(tmp_path, rows, cols):
    world = rows * cols
    mp.spawn(_gpu_worker, args=(world, _free_port(), rows, cols, tmp_path), nprocs=world, join=True)
    for rank in range(world):
        err = json.loads((tmp_path / f"r{rank}.json").read_text())
        assert err["ab"] < 1e-4 and err["abt"] < 1e-4 and err["atb"] < 1e-4, err
        assert err["loss"] < 1e-3 and err["grads"] < 2e-2, err
