"""Megatron-style 1D tensor-parallel layer: the paper's comparison baseline
(drop-in for summagrid baseline.py:40-224), on the same sm_100a kernels.

Every position holds the whole [b*s, h] activations (replicated), a 1/p column
slice of the first weight of each sub-layer (whole heads for attention: the QKV
columns are interleaved per position, layers.py:87-115) and a 1/p row slice of
the second; the two partial outputs per layer are summed by an all-reduce over
all p positions (NCCL world all-reduce on the dist backend, a position-ordered
device fold on the single-GPU mesh). Layer norms and the residual / bias adds
run replicated with no communication. Forward: 2 all-reduces of b*s*h scalars;
backward: 2 more, as in the reference.

Numerics follow the reference layer on identical gathered parameters (bf16
operands, fp32 accumulate here); only the partition and the traffic differ.
"""

from __future__ import annotations

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigError
from .layers import ModelConfig, attention_core_backward, attention_core_forward, deinterleave_qkv, interleave_qkv
from .membuf import Workspace, padded_empty
from .mesh import Mesh

BF16, F32 = torch.bfloat16, torch.float32


def _dev_tensor(a, dtype, device) -> torch.Tensor:
    a = np.asarray(a, dtype=np.float64)
    t = padded_empty(a.shape, dtype, device)
    t.copy_(torch.as_tensor(a, dtype=F32).to(dtype))
    return t


class Baseline1DLayer:
    """One transformer layer in the 1D partition over the mesh's p positions (baseline.py:40)."""

    def __init__(self, mesh: Mesh, cfg: ModelConfig, layer_params: dict) -> None:
        p = mesh.p
        if cfg.n % p:
            raise ConfigError(f"1D partition needs heads n={cfg.n} divisible by p={p}")
        if cfg.h % p:
            raise ConfigError(f"1D partition needs hidden h={cfg.h} divisible by p={p}")
        self.mesh = mesh
        self.cfg = cfg
        dev = mesh.device()
        h, hp = cfg.h, cfg.h // p
        g = {k: np.asarray(v, dtype=np.float64) for k, v in layer_params.items()}
        w_qkv_il, b_qkv_il = interleave_qkv(g["w_qkv"], p), interleave_qkv(g["b_qkv"], p)
        self.shards: list = [None] * p
        for d in mesh.local_devs:
            self.shards[d] = {
                "w_qkv": _dev_tensor(w_qkv_il[:, d * 3 * hp:(d + 1) * 3 * hp], BF16, dev),
                "b_qkv": _dev_tensor(b_qkv_il[d * 3 * hp:(d + 1) * 3 * hp], F32, dev),
                "w_dense": _dev_tensor(g["w_dense"][d * hp:(d + 1) * hp, :], BF16, dev),
                "w1": _dev_tensor(g["w1"][:, d * 4 * hp:(d + 1) * 4 * hp], BF16, dev),
                "b1": _dev_tensor(g["b1"][d * 4 * hp:(d + 1) * 4 * hp], F32, dev),
                "w2": _dev_tensor(g["w2"][d * 4 * hp:(d + 1) * 4 * hp, :], BF16, dev),
            }
        # replicated parameters
        self.rep = {k: _dev_tensor(g[k], F32, dev) for k in ("b_dense", "b2", "ln1_gamma", "ln1_beta", "ln2_gamma",
                                                              "ln2_beta")}
        self._h = h

    # ---------------------------------------------------------------- helpers
    def _ln(self, x, gamma, beta, ws, dev):
        rows = x.shape[0]
        y = ws.empty(dev, (rows, self._h), "replicated", dtype=BF16)
        mean = ws.empty(dev, (rows,), "free", dtype=F32)
        rstd = ws.empty(dev, (rows,), "free", dtype=F32)
        K.ln_fwd(x, None, self._h, self.cfg.eps, gamma, beta, y, mean, rstd)
        return y, (x, mean, rstd, gamma)

    def _ln_bwd(self, dout, ln, resid, ws, dev):
        """(dx = resid + LN'(dout), dgamma, dbeta, colsum(dx)) for full local rows."""
        x, mean, rstd, gamma = ln
        rows = x.shape[0]
        stats = ws.empty(dev, (rows, 2), "free", dtype=F32, pad=False)
        K.ln_bwd_stats(dout, x, mean, rstd, gamma, stats)
        dx = ws.empty(dev, (rows, self._h), "replicated", dtype=F32)
        dx16 = ws.empty(dev, (rows, self._h), "free", dtype=BF16)
        gb = torch.zeros(3, self._h, device=x.device)
        K.ln_bwd(dout, x, mean, rstd, gamma, stats, self._h, resid, dx, dx16, gb[0], gb[1], gb[2])
        return dx, dx16, gb

    def _all_reduce(self, parts: list, tag: str) -> torch.Tensor:
        self.mesh.allreduce_all(parts, tag=tag)
        return parts[self.mesh.local_devs[0]]

    # ---------------------------------------------------------------- forward
    def forward(self, x, ws: Workspace):
        """x: the replicated [b*s, h] input (host array or device tensor); returns the
        replicated output (device fp32) and the saved state (baseline.py:93-164)."""
        mesh, cfg = self.mesh, self.cfg
        p, bs = mesh.p, cfg.b * cfg.s
        dev0 = mesh.local_devs[0]
        device = mesh.device()
        x = torch.as_tensor(np.asarray(x) if not isinstance(x, torch.Tensor) else x).to(device=device, dtype=F32)
        xr = ws.empty(dev0, (bs, cfg.h), "replicated", dtype=F32)
        xr.copy_(x)
        a1, ln1 = self._ln(xr, self.rep["ln1_gamma"], self.rep["ln1_beta"], ws, dev0)
        n_loc, hp = cfg.n // p, cfg.h // p
        h, att_macs = cfg.h, cfg.b * n_loc * cfg.s * cfg.s * cfg.head_dim
        # per-position multiply-accumulates, as the reference's local_matmul / add_macs charge them
        mesh.add_macs_all(bs * h * 3 * hp + 2 * att_macs + bs * hp * h + bs * h * 4 * hp + bs * 4 * hp * h)
        saved = {"ln1": ln1, "a1": a1, "dev": [None] * p}
        parts = [None] * p
        for d in mesh.local_devs:
            sh = self.shards[d]
            qkv = ws.empty(d, (bs, 3 * hp), "forward", dtype=BF16)
            K.gemm(a1, sh["w_qkv"], qkv, bias=sh["b_qkv"])
            ctx = ws.empty(d, (bs, hp), "forward", dtype=BF16)
            probs, lse = attention_core_forward(cfg, cfg.b, n_loc, qkv, ctx, ws, d, device)
            parts[d] = ws.empty(d, (bs, cfg.h), "workspace", dtype=F32)
            K.gemm(ctx, sh["w_dense"], parts[d])
            saved["dev"][d] = {"qkv": qkv, "ctx": ctx, "probs": probs, "lse": lse}
        att = self._all_reduce(parts, "baseline")
        y1 = ws.empty(dev0, (bs, cfg.h), "replicated", dtype=F32)
        K.epilogue(att, y1, bias=self.rep["b_dense"], c=xr)
        a2, ln2 = self._ln(y1, self.rep["ln2_gamma"], self.rep["ln2_beta"], ws, dev0)
        saved.update(y1=y1, ln2=ln2, a2=a2)
        parts = [None] * p
        for d in mesh.local_devs:
            sh = self.shards[d]
            mid = ws.empty(d, (bs, 4 * hp), "forward", dtype=BF16)
            act = ws.empty(d, (bs, 4 * hp), "forward", dtype=BF16)
            K.gemm(a2, sh["w1"], act, bias=sh["b1"], act=K.ACT_GELU, aux=mid)
            parts[d] = ws.empty(d, (bs, cfg.h), "workspace", dtype=F32)
            K.gemm(act, sh["w2"], parts[d])
            saved["dev"][d].update(mid=mid, act=act)
        mlp = self._all_reduce(parts, "baseline")
        out = ws.empty(dev0, (bs, cfg.h), "replicated", dtype=F32)
        K.epilogue(mlp, out, bias=self.rep["b2"], c=y1)
        return out, saved

    # ---------------------------------------------------------------- backward
    def backward(self, dy, saved: dict, ws: Workspace, host_grads: bool = True):
        """(dx, standard-layout parameter gradients as host arrays) (baseline.py:166-220);
        ``host_grads=False`` keeps them as this process's device shards (timing)."""
        mesh, cfg = self.mesh, self.cfg
        p, bs = mesh.p, cfg.b * cfg.s
        n_loc, hp = cfg.n // p, cfg.h // p
        dev0 = mesh.local_devs[0]
        device = mesh.device()
        dyf = ws.empty(dev0, (bs, cfg.h), "replicated", dtype=F32)
        dyf.copy_(torch.as_tensor(np.asarray(dy) if not isinstance(dy, torch.Tensor) else dy).to(device, F32))
        dy16 = ws.empty(dev0, (bs, cfg.h), "free", dtype=BF16)
        dy16.copy_(dyf)
        h, att_macs = cfg.h, cfg.b * n_loc * cfg.s * cfg.s * cfg.head_dim
        mesh.add_macs_all(4 * bs * h * 4 * hp + 2 * bs * hp * h + 4 * att_macs + 2 * bs * 3 * hp * h)
        b2_grad = torch.zeros(cfg.h, device=device)
        K.colsum(dyf, b2_grad, accumulate=True)
        dw1, db1, dw2 = [None] * p, [None] * p, [None] * p
        parts = [None] * p
        for d in mesh.local_devs:
            sh, sv = self.shards[d], saved["dev"][d]
            dw2[d] = torch.empty(4 * hp, cfg.h, device=device)
            K.gemm(sv["act"].t(), dy16, dw2[d])
            dmid = ws.empty(d, (bs, 4 * hp), "backward", dtype=BF16)
            db1[d] = torch.zeros(4 * hp, device=device)
            K.gemm(dy16, sh["w2"].t(), dmid, act=K.ACT_DGELU, aux=sv["mid"], colsum=db1[d])
            dw1[d] = torch.empty(cfg.h, 4 * hp, device=device)
            K.gemm(saved["a2"].t(), dmid, dw1[d])
            parts[d] = ws.empty(d, (bs, cfg.h), "workspace", dtype=F32)
            K.gemm(dmid, sh["w1"].t(), parts[d])
        da2 = self._all_reduce(parts, "baseline")
        dy1, dy1_16, gb2 = self._ln_bwd(da2, saved["ln2"], dyf, ws, dev0)
        dwqkv, dbqkv, dwd = [None] * p, [None] * p, [None] * p
        parts = [None] * p
        for d in mesh.local_devs:
            sh, sv = self.shards[d], saved["dev"][d]
            dwd[d] = torch.empty(hp, cfg.h, device=device)
            K.gemm(sv["ctx"].t(), dy1_16, dwd[d])
            dctx = ws.empty(d, (bs, hp), "backward", dtype=BF16)
            K.gemm(dy1_16, sh["w_dense"].t(), dctx)
            dbqkv[d] = torch.zeros(3 * hp, device=device)
            qkv = sv["qkv"]
            dqkv = attention_core_backward(
                cfg, cfg.b, n_loc, qkv, sv["ctx"], dctx, sv["lse"],
                lambda qkv=qkv, sv=sv: sv["probs"] if sv["probs"] is not None else _rebuild_probs(cfg, n_loc, qkv),
                ws, d, device, dbqkv[d])
            dwqkv[d] = torch.empty(cfg.h, 3 * hp, device=device)
            K.gemm(saved["a1"].t(), dqkv, dwqkv[d])
            parts[d] = ws.empty(d, (bs, cfg.h), "workspace", dtype=F32)
            K.gemm(dqkv, sh["w_qkv"].t(), parts[d])
        da1 = self._all_reduce(parts, "baseline")
        dx, _, gb1 = self._ln_bwd(da1, saved["ln1"], dy1, ws, dev0)
        if not host_grads:
            return dx, {"w_qkv": dwqkv, "b_qkv": dbqkv, "w_dense": dwd, "w1": dw1, "b1": db1, "w2": dw2,
                        "b2": b2_grad, "ln": (gb1, gb2)}

        def host(ts, axis):
            return np.concatenate(_gather_parts(mesh, ts), axis=axis)

        grads = {
            "w_qkv": deinterleave_qkv(host(dwqkv, 1), p),
            "b_qkv": deinterleave_qkv(host(dbqkv, 0), p),
            "w_dense": host(dwd, 0),
            "b_dense": gb2[2].double().cpu().numpy(),
            "w1": host(dw1, 1),
            "b1": host(db1, 0),
            "w2": host(dw2, 0),
            "b2": b2_grad.double().cpu().numpy(),
            "ln1_gamma": gb1[0].double().cpu().numpy(),
            "ln1_beta": gb1[1].double().cpu().numpy(),
            "ln2_gamma": gb2[0].double().cpu().numpy(),
            "ln2_beta": gb2[1].double().cpu().numpy(),
        }
        return dx, grads


def _rebuild_probs(cfg: ModelConfig, n_loc: int, qkv):
    from .layers import _probs_core

    return _probs_core(cfg, cfg.b, n_loc, qkv, qkv.device)


def _gather_parts(mesh: Mesh, parts: list) -> list:
    """Per-position shards as host float64 arrays in position order (all processes on dist)."""
    if mesh.is_local:
        return [t.detach().double().cpu().numpy() for t in parts]
    import torch.distributed as dist

    mine = parts[mesh.my_flat].detach().double().cpu().numpy()
    out = [None] * mesh.p
    dist.all_gather_object(out, (mesh.my_flat, mine))
    res = [None] * mesh.p
    for f, a in out:
        res[f] = a
    return res
