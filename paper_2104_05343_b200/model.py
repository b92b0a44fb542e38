"""End-to-end 2D model: embedding -> N pre-norm layers -> tied lm-head -> mean CE.

Drop-in for summagrid model.py:97-424 (MeshModel, init_global_params,
run_loss_and_grads). Parameters live on the mesh as fp32 masters with bf16
twins for the tensor-core GEMMs; the table is padded with zero rows to
v_padded and stored in the SUMMA weight layout; the QKV weight is
column-interleaved per mesh column and de-interleaved on gather, so loss and
gathered gradients are independent of the mesh shape.

``train_step`` is the sync-free training step (forward, backward, SGD) the
bench times and captures into a CUDA graph; ``forward`` / ``backward`` keep
the reference's signatures.
"""

from __future__ import annotations

import math
import struct
from dataclasses import dataclass
from typing import Optional

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigError, ShapeError
from .layers import (
    LayerGrads,
    LayerParams,
    ModelConfig,
    RowHostedVector,
    TransformerLayer,
    _device_ids,
    cross_entropy_backward,
    cross_entropy_forward,
    deinterleave_qkv,
    embedding_backward,
    embedding_forward,
    interleave_qkv,
    sgd_matrix,
    sgd_vector,
)
from .membuf import CheckpointStore, Workspace, checkpointed_backward, checkpointed_forward, clone_to_conjunction, \
    padded_empty
from .mesh import Mesh
from .summa import BF16, F32, ShardedMatrix, as_bf16, gather, scatter, summa_ab, summa_abt, summa_atb

_LAYER_KEYS = ("ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_dense", "b_dense", "ln2_gamma", "ln2_beta", "w1", "b1",
               "w2", "b2")
_MATS = ("w_qkv", "w_dense", "w1", "w2")


def param_declaration_order(cfg: ModelConfig) -> list[str]:
    """Parameter names in the reference's declaration order (model.py:71-79)."""
    names = ["table"]
    for i in range(cfg.num_layers):
        names += [f"layers.{i}.{k}" for k in _LAYER_KEYS]
    return names


def param_shape(cfg: ModelConfig, name: str) -> tuple[int, ...]:
    h = cfg.h
    base = name.rsplit(".", 1)[-1]
    return {"table": (cfg.v, h), "w_qkv": (h, 3 * h), "b_qkv": (3 * h,), "w_dense": (h, h), "w1": (h, 4 * h),
            "b1": (4 * h,), "w2": (4 * h, h)}.get(base, (h,))


# ---------------------------------------------------------------- checkpoint file
# The reference's on-disk model format (model.py:64-79, 431-462): little-endian
# header of eight u64 (magic, version, b, s, h, n, v, num_layers), u64 classifier
# flag, f64 eps, then every parameter as f64 row-major in declaration order.
CKPT_MAGIC = 0x5347524944434B50
CKPT_VERSION = 1
_CKPT_HEADER = struct.Struct("<8QQd")


def _ckpt_names(cfg: ModelConfig, classifier: bool) -> list[str]:
    return param_declaration_order(cfg) + (["cls_w"] if classifier else [])


def _ckpt_shape(cfg: ModelConfig, name: str) -> tuple[int, ...]:
    return (cfg.h, 2) if name == "cls_w" else param_shape(cfg, name)


def save_checkpoint(path, cfg: ModelConfig, global_params: dict, classifier: bool = False) -> None:
    """Write ``global_params`` (host arrays, standard layout) in the reference's
    binary checkpoint format (model.py:431-445); ShapeError on a wrong shape."""
    with open(path, "wb") as f:
        f.write(_CKPT_HEADER.pack(CKPT_MAGIC, CKPT_VERSION, cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers,
                                  1 if classifier else 0, float(cfg.eps)))
        for name in _ckpt_names(cfg, classifier):
            arr = np.ascontiguousarray(np.asarray(global_params[name]), dtype="<f8")
            if arr.shape != _ckpt_shape(cfg, name):
                raise ShapeError(f"{name}: expected {_ckpt_shape(cfg, name)}, got {arr.shape}")
            f.write(arr.tobytes())


def load_checkpoint(path) -> tuple[ModelConfig, dict, bool]:
    """(cfg, host f64 parameters, classifier flag) of a reference checkpoint file
    (model.py:448-462); ConfigError on a bad magic / version or a truncated file."""
    with open(path, "rb") as f:
        head = f.read(_CKPT_HEADER.size)
        if len(head) != _CKPT_HEADER.size:
            raise ConfigError("checkpoint file truncated (header)")
        magic, version, b, s, h, n, v, layers, cls_flag, eps = _CKPT_HEADER.unpack(head)
        if magic != CKPT_MAGIC:
            raise ConfigError(f"not a model checkpoint (bad magic {magic:#x})")
        if version != CKPT_VERSION:
            raise ConfigError(f"unsupported checkpoint version {version}")
        cfg = ModelConfig(b=b, s=s, h=h, n=n, v=v, num_layers=layers, eps=eps)
        classifier = bool(cls_flag)
        params = {}
        for name in _ckpt_names(cfg, classifier):
            shape = _ckpt_shape(cfg, name)
            count = int(np.prod(shape))
            raw = f.read(8 * count)
            if len(raw) != 8 * count:
                raise ConfigError(f"checkpoint file truncated at {name}")
            params[name] = np.frombuffer(raw, dtype="<f8").reshape(shape).copy()
    return cfg, params, classifier


def init_global_params(cfg: ModelConfig, seed: int, classifier: bool = False) -> dict[str, np.ndarray]:
    """Host float64 parameters, identical for every mesh (model.py:97-119).

    PCG64(seed) draws U[-1/sqrt(h), 1/sqrt(h)) in the order table, then per
    layer w_qkv, w_dense, w1, w2; vectors start at identity (gamma=1, rest 0).
    """
    rng = np.random.Generator(np.random.PCG64(seed))
    lim = 1.0 / math.sqrt(cfg.h)
    out = {"table": rng.uniform(-lim, lim, size=(cfg.v, cfg.h))}
    for i in range(cfg.num_layers):
        pre = f"layers.{i}."
        for name in _LAYER_KEYS:
            shape = param_shape(cfg, name)
            if name in _MATS:
                out[pre + name] = rng.uniform(-lim, lim, size=shape)
            else:
                out[pre + name] = (np.ones if name.endswith("gamma") else np.zeros)(shape)
    if classifier:  # drawn after every layer (model.py:116-117)
        out["cls_w"] = rng.uniform(-lim, lim, size=(cfg.h, 2))
    return out


@dataclass
class ModelGrads:
    table: ShardedMatrix
    layers: list
    cls_w: Optional[list] = None


@dataclass
class ModelSaved:
    tokens: object
    labels: object
    x_final: ShardedMatrix
    ce_ctx: object
    layer_saves: Optional[list] = None
    store: Optional[CheckpointStore] = None
    ids: Optional[list] = None
    cls_ctx: Optional[dict] = None


def _with_twin(m: ShardedMatrix) -> ShardedMatrix:
    """Attach the bf16 GEMM copy of an fp32 master; on a peer-memory mesh both live in
    the symmetric arena (remote reduce-adds into the master, panel pulls of the twin)."""
    if m.dtype == BF16:
        raise ConfigError("masters must be fp32")
    if m.mesh.peer is not None:
        from .membuf import copy_block

        blocks = [None if b is None else copy_block(m.mesh.persistent_empty(tuple(b.shape), BF16), b)
                  for b in m.blocks]
        m.bf16_twin = ShardedMatrix(m.mesh, m.global_rows, m.global_cols, blocks, m.layout)
    else:
        m.bf16_twin = as_bf16(m)
    return m


class MeshModel:
    """Distributed transformer bound to one mesh (model.py:152-411)."""

    def __init__(self, mesh: Mesh, cfg: ModelConfig, global_params: dict | None = None, classifier: bool = False,
                 skip_dead_recompute: bool = False, *, seed: int = 0, logits_dtype: torch.dtype = BF16) -> None:
        cfg.validate_mesh(mesh)
        self.mesh = mesh
        self.cfg = cfg
        self.classifier = classifier
        self.logits_dtype = logits_dtype
        self._bad_ids: torch.Tensor | None = None  # device-side id range-check flag
        c = mesh.c
        v_pad = cfg.v_padded(mesh)
        if global_params is None:
            self.table = _device_random(mesh, v_pad, cfg.h, cfg, seed, rows_real=cfg.v)
        else:
            tab = np.asarray(global_params["table"], dtype=np.float64)
            if v_pad != cfg.v:
                tab = np.vstack([tab, np.zeros((v_pad - cfg.v, cfg.h))])
            self.table = _with_twin(scatter(tab, mesh, layout="weight", persistent=True))
        self.layers: list[TransformerLayer] = []
        for i in range(cfg.num_layers):
            pre = f"layers.{i}."
            if global_params is None:
                kw = {name: _device_random(mesh, *param_shape(cfg, name), cfg, seed * 1000 + 10 * i + k)
                      for k, name in enumerate(_MATS)}
                kw["w_qkv"] = kw["w_qkv"]  # random init is layout-agnostic
                vec = {name: RowHostedVector.split(
                    (np.ones if name.endswith("gamma") else np.zeros)(param_shape(cfg, name)), c, mesh=mesh)
                    for name in _LAYER_KEYS if name not in _MATS}
            else:
                g = global_params
                kw = {"w_qkv": _with_twin(scatter(interleave_qkv(np.asarray(g[pre + "w_qkv"]), c), mesh,
                                                  layout="weight", persistent=True)),
                      "w_dense": _with_twin(scatter(g[pre + "w_dense"], mesh, layout="weight", persistent=True)),
                      "w1": _with_twin(scatter(g[pre + "w1"], mesh, layout="weight", persistent=True)),
                      "w2": _with_twin(scatter(g[pre + "w2"], mesh, layout="weight", persistent=True))}
                vec = {name: RowHostedVector.split(
                    interleave_qkv(np.asarray(g[pre + name]), c) if name == "b_qkv" else g[pre + name], c, mesh=mesh)
                    for name in _LAYER_KEYS if name not in _MATS}
            params = LayerParams(**kw, **vec)
            self.layers.append(TransformerLayer(mesh, cfg, params, skip_dead_recompute=skip_dead_recompute))
        # position-0 binary classifier head (model.py:123-131, 185-188): the [h, 2]
        # weight split by rows over the mesh columns, a replica per column
        self.cls_w: list | None = None
        self.cls_w16: list | None = None
        if classifier:
            w = (np.asarray(global_params["cls_w"], dtype=np.float64) if global_params is not None
                 else np.random.default_rng(seed + 7).uniform(-1 / math.sqrt(cfg.h), 1 / math.sqrt(cfg.h), (cfg.h, 2)))
            hb = cfg.h // c
            self.cls_w, self.cls_w16 = [None] * c, [None] * c
            for j in range(c):
                if not mesh.is_local and mesh.my_flat % c != j:
                    continue
                self.cls_w[j] = padded_empty((hb, 2), F32, mesh.device())
                self.cls_w[j].copy_(torch.as_tensor(w[j * hb:(j + 1) * hb], dtype=F32))
                self.cls_w16[j] = padded_empty((hb, 2), BF16, mesh.device())
                self.cls_w16[j].copy_(self.cls_w[j])

    # ------------------------------------------------------------------ workspace
    def workspace_capacities(self, checkpointing: bool = True, eager_update: bool = False) -> dict:
        """Planned per-position scalars per arena category (the reference's plan,
        model.py:197-222, restated for this build's allocations). Same as the reference:
        forward 9 bsh/p per layer (QKV 3, attention out 1, MLP pre-activation 4, MLP out 1;
        + the embedding output without checkpointing), backward 7 bsh/p, conjunction
        bsh/p. Different, because of the fused kernels: the flash path keeps the row
        log-sum-exp (b n s / p) instead of P; vector gradients 13 h/c per layer plus the
        last layer's b2 gradient formed by the lm-head product (h/c); with eager SGD on a
        local / peer-memory mesh the weight gradients never exist (updated inside their
        products); the tied table gradient is one set of blocks (the embedding backward
        accumulates into it); the per-product workspace is _workspace_plan's."""
        from .layers import flash_ok

        cfg, mesh = self.cfg, self.mesh
        r, c, p = mesh.r, mesh.c, mesh.p
        rows, hb, vb = cfg.b * cfg.s // r, cfg.h // c, cfg.v_padded(mesh) // c
        bsh_p = rows * hb
        lse = (cfg.b // r) * (cfg.n // c) * cfg.s if flash_ok(cfg) else 0
        fwd_layer = 9 * bsh_p + lse
        mats, vecs = 12 * cfg.h * cfg.h // p, 13 * hb
        fused = mesh.is_local or mesh.peer is not None
        cls = 2 * hb if self.classifier else 0
        if eager_update and checkpointing:
            param_grad = vecs + hb + cls + (0 if fused else mats)
        else:
            param_grad = max(cfg.num_layers, 1) * (mats + vecs) + hb + cls
        return {"workspace": self._workspace_plan(),
                "forward": fwd_layer if checkpointing else cfg.num_layers * fwd_layer + bsh_p,
                "backward": 7 * bsh_p, "param_grad": param_grad, "param_grad_tied": (c // r) * vb * hb,
                "conjunction": bsh_p, "free": None, "replicated": None}

    def _workspace_plan(self) -> int:
        """Largest per-product "workspace" use (reset at every SUMMA product, summa.py).

        local mesh: one step needs none; c > 1 stages the fp32 sum of a product whose
        epilogue needs the complete sum (bf16 QKV / fc1 / dctx / dAct outputs, the bf16
        logits): max(4 bsh/p, bs v/(r c)). dist: two receive slots per broadcast operand,
        plus (collective reduce) two partial-sum slots and the fold accumulator; with
        peer memory the partial sums go to the destination's symmetric accumulator."""
        cfg, mesh = self.cfg, self.mesh
        r, c = mesh.r, mesh.c
        R, hb, vb = cfg.b * cfg.s // r, cfg.h // c, cfg.v_padded(mesh) // c
        bf16_logits = self.logits_dtype == BF16
        if mesh.is_local:
            return 0 if c == 1 else max(4 * R * hb, R * vb if bf16_logits else 0)
        peer = mesh.peer is not None
        # (m_b, k_b, n_b, epilogue needs the full sum) per product of the step
        ab = [(R, hb, 3 * hb, True), (R, hb, hb, False), (R, hb, 4 * hb, True), (R, 4 * hb, hb, False),
              (R, vb, hb, True)]
        abt = [(R, hb, hb), (R, hb, 4 * hb), (R, 3 * hb, hb), (R, 4 * hb, hb), (R, hb, vb)]
        atb = [(hb, R, hb), (4 * hb, R, hb), (hb, R, 4 * hb), (hb, R, 3 * hb), (vb, R, hb)]
        need = [2 * m * k + 2 * k * n + (m * n if full else 0) for m, k, n, full in ab]
        need += [2 * n * k + (0 if peer else 3 * m * n) for m, k, n in abt]
        need += [2 * t * m + (0 if peer else 2 * m * n) for m, t, n in atb]
        need.append(vb * hb)  # embedding backward staging (column reduce)
        return max(need)

    def make_workspace(self, checkpointing: bool = True, eager_update: bool = False, merge_fwd_bwd: bool = False,
                       planned: bool = False) -> Workspace:
        """Per-position arenas (membuf.py:74-127); ``planned`` enforces
        workspace_capacities (BufferOverflowError on overflow, model.py:219-222)."""
        caps = self.workspace_capacities(checkpointing, eager_update) if planned else None
        return Workspace(self.mesh.p, capacities=caps, merge_fwd_bwd=merge_fwd_bwd, device=self.mesh.device())

    # ------------------------------------------------------------------ forward / backward
    def forward(self, tokens, labels, ws: Workspace, store: CheckpointStore | None = None, cls_labels=None, *,
                return_tensor: bool = False):
        """Loss (python float, or a device tensor with return_tensor) and saved state (model.py:296-324)."""
        cfg = self.cfg
        if tuple(tokens.shape) != (cfg.b, cfg.s):
            raise ShapeError(f"tokens must be [{cfg.b}, {cfg.s}], got {tuple(tokens.shape)}")
        if self.classifier and cls_labels is None:
            raise ConfigError("classifier enabled but cls_labels missing")
        ws.reset_all("forward")
        ws.reset_all("free")
        ids, label_ids = self._validated_ids(tokens, labels)
        x = embedding_forward(tokens, self.table, cfg, ws, out_category="forward", ids=ids)
        layer_saves = None
        if store is not None:
            x = checkpointed_forward(self.layers, x, store, ws)
        else:
            layer_saves = []
            for layer in self.layers:
                x, saved = layer.forward(x, ws)
                layer_saves.append(saved)
        if getattr(x, "bf16_twin", None) is None and x.dtype != BF16:
            x.bf16_twin = as_bf16(x)  # one cast, shared by the logits and the table-gradient products
        with K.tagged("logits"):
            logits = summa_abt(x, self.table, ws, tag="lmhead", out_dtype=self.logits_dtype)
        loss, ce_ctx = cross_entropy_forward(logits, labels, cfg, ws, return_tensor=return_tensor,
                                             label_ids=label_ids)
        if not return_tensor:
            self.check_inputs()  # the loss read-back already synchronised
        cls_ctx = None
        if self.classifier:
            cls_loss, cls_ctx = self._cls_forward(x, cls_labels, ws)
            loss = loss + (cls_loss if return_tensor else float(cls_loss.item()))
        return loss, ModelSaved(tokens=tokens, labels=labels, x_final=x, ce_ctx=ce_ctx, layer_saves=layer_saves,
                                store=store, ids=ids, cls_ctx=cls_ctx)

    # ------------------------------------------------------------------ input validation
    def _validated_ids(self, tokens, labels):
        """Per-position device ids of tokens and labels, range-checked against v
        (layers.py:164-165, 552-553): host arrays on the host (ConfigError now),
        device tensors by a device kernel into ``self._bad_ids`` (no host sync in
        the step; ConfigError at the next check_inputs / float loss read-back)."""
        from .layers import _check_ids

        if self._bad_ids is None:
            self._bad_ids = torch.zeros(1, dtype=torch.int32, device=self.mesh.device())
        for arr, what in ((tokens, "token ids"), (labels, "labels")):
            _check_ids(arr, self.cfg.v, what, flag=self._bad_ids if isinstance(arr, torch.Tensor) and arr.is_cuda
                       else None)
        return _device_ids(self.mesh, tokens), _device_ids(self.mesh, labels)

    def check_inputs(self) -> None:
        """Raise ConfigError if a device-side id check of an earlier step failed (one
        host synchronisation); clears the flag."""
        if self._bad_ids is not None and int(self._bad_ids.item()):
            self._bad_ids.zero_()
            raise ConfigError(f"token ids / labels must lie in [0, {self.cfg.v})")

    def backward(self, saved: ModelSaved, ws: Workspace, upstream: float = 1.0, eager_update: bool = False,
                 lr: float = 0.0, *, _fused_sgd_lr: float | None = None) -> ModelGrads:
        """Gradients of every parameter (model.py:326-354); the tied table gets
        lm-head dW plus the embedding scatter-add, accumulated in place."""
        cfg, mesh = self.cfg, self.mesh
        dl = cross_entropy_backward(saved.ce_ctx, mesh, ws, upstream, in_place=True)
        dlogits = ShardedMatrix(mesh, cfg.b * cfg.s, cfg.v_padded(mesh), dl)
        from .layers import new_colsum_parts

        if self.classifier:
            # the head adds into dx after the product: its bf16 twin and column sums are
            # formed later, by the layer (_bf16_of / bias_add_backward)
            with K.tagged("dx_lmhead"):
                dx = summa_ab(dlogits, self.table, ws, out_category="conjunction", tag="lmhead", out_dtype=F32)
        else:
            parts = new_colsum_parts(mesh, ws, cfg.h // mesh.c)  # last layer's b2 gradient, fused
            with K.tagged("dx_lmhead"):
                dx = summa_ab(dlogits, self.table, ws, out_category="conjunction", tag="lmhead", out_dtype=F32,
                              want_bf16=True, colsum=parts)
            dx.colsum_parts = parts
        with K.tagged("dw_table"):
            table_grad = summa_atb(dlogits, saved.x_final, ws, out_category="param_grad_tied", tag="lmhead")
        cls_w_grad = self._cls_backward(saved.cls_ctx, dx, ws, upstream) if self.classifier else None
        if saved.store is not None:
            dx0, layer_grads = checkpointed_backward(self.layers, dx, saved.store, ws, eager_update=eager_update,
                                                     lr=lr)
        else:
            # the reference's non-checkpointed backward ignores eager_update: it returns every
            # layer gradient and leaves the parameters alone (model.py:343-351); the fused
            # update is train_step's (``_fused_sgd_lr``)
            layer_grads = [None] * len(self.layers)
            dy = dx
            for li in reversed(range(len(self.layers))):
                ws.reset_all("backward")
                if _fused_sgd_lr is not None and getattr(self.layers[li], "fused_sgd", False):
                    dy, g = self.layers[li].backward(dy, saved.layer_saves[li], ws, lr=_fused_sgd_lr)
                else:
                    dy, g = self.layers[li].backward(dy, saved.layer_saves[li], ws)
                if _fused_sgd_lr is not None:
                    self.layers[li].apply_sgd(g, _fused_sgd_lr)
                else:
                    layer_grads[li] = g
            dx0 = dy
        embedding_backward(dx0, saved.tokens, self.table, cfg, ws, ids=saved.ids, accumulate_into=table_grad)
        return ModelGrads(table=table_grad, layers=layer_grads, cls_w=cls_w_grad)

    # ------------------------------------------------------------------ classifier branch
    def _cls_x0(self, x: ShardedMatrix, dev: int) -> torch.Tensor:
        """Rows at sequence position 0 of a position's [b_loc*s, h/c] block (a strided view)."""
        blk = x.blocks[dev]
        b_loc = self.cfg.b // self.mesh.r
        return torch.as_strided(blk, (b_loc, blk.shape[1]), (self.cfg.s * blk.stride(0), 1))

    def _cls_forward(self, x_final: ShardedMatrix, cls_labels, ws: Workspace):
        """Position-0 binary classifier loss (model.py:238-276): partial logits x0 W_j
        row-all-reduced, softmax cross entropy, mean over the b sequences."""
        mesh, cfg = self.mesh, self.cfg
        b_loc, hb, c = cfg.b // mesh.r, cfg.h // mesh.c, mesh.c
        labels = torch.as_tensor(np.asarray(cls_labels.cpu() if isinstance(cls_labels, torch.Tensor) else cls_labels),
                                 dtype=torch.int64)
        if labels.shape != (cfg.b,):
            raise ShapeError(f"cls_labels must be [{cfg.b}], got {tuple(labels.shape)}")
        if labels.numel() and (int(labels.min()) < 0 or int(labels.max()) > 1):
            raise ConfigError("cls_labels must lie in [0, 2)")
        x0, logits, labs = [None] * mesh.p, [None] * mesh.p, [None] * mesh.p
        for dev in mesh.local_devs:
            x0[dev] = ws.empty(dev, (b_loc, hb), "free", dtype=BF16)
            K.epilogue(self._cls_x0(x_final, dev), x0[dev])
            logits[dev] = ws.empty(dev, (b_loc, 2), "free", dtype=F32)
            K.gemm(x0[dev], self.cls_w16[dev % c], logits[dev])
            i = dev // c
            labs[dev] = labels[i * b_loc:(i + 1) * b_loc].to(mesh.device())
        mesh.allreduce_row(logits, tag="classifier")
        gmax, packed, part = [None] * mesh.p, [None] * mesh.p, [None] * mesh.p
        for dev in mesh.local_devs:
            lmax = ws.empty(dev, (b_loc,), "free", dtype=F32)
            gmax[dev] = ws.empty(dev, (b_loc,), "free", dtype=F32)
            packed[dev] = ws.empty(dev, (b_loc, 2), "free", dtype=F32, pad=False)
            K.xent_local(logits[dev], 2, labs[dev], 0, lmax, gmax[dev], packed[dev])
            rows = ws.empty(dev, (b_loc,), "free", dtype=F32)
            part[dev] = ws.empty(dev, (1,), "free", dtype=F32)
            K.xent_loss(gmax[dev], packed[dev], rows, part[dev])
        mesh.allreduce_col(part, tag="classifier")
        loss = part[mesh.local_devs[0]] / cfg.b
        return loss, {"x0": x0, "logits": logits, "labels": labs, "gmax": gmax, "packed": packed}

    def _cls_backward(self, ctx: dict, dx_final: ShardedMatrix, ws: Workspace, upstream: float = 1.0) -> list:
        """dW_j = x0^T dlogits (column-reduced to each column's shard) and dx0 =
        dlogits W_j^T added into dx at sequence position 0 (model.py:278-292)."""
        mesh, cfg = self.mesh, self.cfg
        b_loc, hb, c = cfg.b // mesh.r, cfg.h // mesh.c, mesh.c
        dw = [None] * mesh.p
        for dev in mesh.local_devs:
            dl = ws.empty(dev, (b_loc, 2), "free", dtype=F32)
            K.xent_bwd(ctx["logits"][dev], 2, ctx["labels"][dev], 0, ctx["gmax"][dev], ctx["packed"][dev],
                       upstream / cfg.b, dl)
            dl16 = ws.empty(dev, (b_loc, 2), "free", dtype=BF16)
            K.epilogue(dl, dl16)
            dw[dev] = ws.empty(dev, (hb, 2), "param_grad", dtype=F32)
            K.gemm(ctx["x0"][dev].t(), dl16, dw[dev])
            dx0 = self._cls_x0(dx_final, dev)
            K.gemm(dl16, self.cls_w16[dev % c].t(), dx0, c=dx0)
        mesh.allreduce_col(dw, tag="classifier")
        shards = [None] * c
        for dev in mesh.local_devs:
            if shards[dev % c] is None:
                shards[dev % c] = dw[dev]
        return shards

    def apply_sgd(self, grads: ModelGrads, lr: float) -> None:
        sgd_matrix(self.table, grads.table, lr)
        for layer, g in zip(self.layers, grads.layers):
            if g is not None:
                layer.apply_sgd(g, lr)
        self._cls_sgd(grads, lr)

    def _cls_sgd(self, grads: ModelGrads, lr: float) -> None:
        if self.cls_w is not None and grads.cls_w is not None:
            K.sgd_multi([(w, w16, g) for w, w16, g in zip(self.cls_w, self.cls_w16, grads.cls_w) if w is not None], lr)

    def train_step(self, tokens, labels, ws: Workspace, lr: float, checkpointing: bool = False,
                   cls_labels=None) -> torch.Tensor:
        """One fwd + bwd + SGD step with no host synchronisation; returns the loss tensor.
        Device token / label ids are range-checked on the device: ``check_inputs()``
        raises ConfigError for a step that saw an out-of-range id."""
        store = CheckpointStore(self.mesh.p) if checkpointing else None
        loss, saved = self.forward(tokens, labels, ws, store=store, return_tensor=True, cls_labels=cls_labels)
        grads = self.backward(saved, ws, eager_update=True, lr=lr, _fused_sgd_lr=None if checkpointing else lr)
        sgd_matrix(self.table, grads.table, lr)
        self._cls_sgd(grads, lr)
        self.mesh.step_boundary()
        return loss

    def infer(self, tokens, labels, ws: Workspace) -> torch.Tensor:
        """Forward-only pass (the paper's inference = b / forward time): the
        reference always computes the CE loss (model.py:296-324); no layer state is kept,
        so memory is one layer's activations plus the logits."""
        cfg = self.cfg
        if tuple(tokens.shape) != (cfg.b, cfg.s):
            raise ShapeError(f"tokens must be [{cfg.b}, {cfg.s}], got {tuple(tokens.shape)}")
        ids, label_ids = self._validated_ids(tokens, labels)
        x = embedding_forward(tokens, self.table, cfg, ws, out_category="forward", ids=ids)
        for layer in self.layers:
            x, _ = layer.forward(x, ws)
        with K.tagged("logits"):
            logits = summa_abt(x, self.table, ws, tag="lmhead", out_dtype=self.logits_dtype)
        loss, _ = cross_entropy_forward(logits, labels, cfg, ws, return_tensor=True, label_ids=label_ids)
        self.mesh.step_boundary()
        return loss

    # ------------------------------------------------------------------ checkpoint file
    def save(self, path) -> None:
        """Gather the parameters and write them in the reference checkpoint format.

        The gather is collective (every process takes part); on the dist backend only
        rank 0 writes, to a temporary file renamed into place, and every rank waits at
        a barrier so no process can read a partially written file."""
        import os

        params = self.gather_params()
        rank0 = self.mesh.is_local or _dist_rank() == 0
        if rank0:
            tmp = f"{os.fspath(path)}.tmp{os.getpid()}"
            save_checkpoint(tmp, self.cfg, params, classifier=self.classifier)
            os.replace(tmp, path)
        if not self.mesh.is_local:
            import torch.distributed as dist

            dist.barrier()

    @classmethod
    def load(cls, path, mesh: Mesh, **kw) -> "MeshModel":
        """A model on ``mesh`` (any shape the dimensions divide) from a checkpoint file."""
        cfg, params, classifier = load_checkpoint(path)
        return cls(mesh, cfg, params, classifier=classifier, **kw)

    # ------------------------------------------------------------------ gather for parity
    def gather_params(self) -> dict[str, np.ndarray]:
        c, cfg = self.mesh.c, self.cfg
        out = {"table": gather(self.table)[:cfg.v]}
        for i, layer in enumerate(self.layers):
            out.update(_gather_layer(f"layers.{i}.", layer.params, c))
        if self.cls_w is not None:
            out["cls_w"] = RowHostedVector([None if w is None else w.reshape(-1) for w in self.cls_w]) \
                .gathered().reshape(cfg.h, 2)
        return out

    def gather_grads(self, grads: ModelGrads) -> dict[str, np.ndarray]:
        c, cfg = self.mesh.c, self.cfg
        out = {"table": gather(grads.table)[:cfg.v]}
        for i, g in enumerate(grads.layers):
            if g is not None:
                out.update(_gather_layer(f"layers.{i}.", g, c))
        if grads.cls_w is not None:
            out["cls_w"] = RowHostedVector([None if w is None else w.reshape(-1) for w in grads.cls_w]) \
                .gathered().reshape(cfg.h, 2)
        return out


def _dist_rank() -> int:
    import torch.distributed as dist

    return dist.get_rank() if dist.is_initialized() else 0


def _gather_layer(pre: str, p, c: int) -> dict:
    out = {}
    for name in _LAYER_KEYS:
        val = getattr(p, name)
        arr = gather(val) if isinstance(val, ShardedMatrix) else val.gathered()
        out[pre + name] = deinterleave_qkv(arr, c) if name in ("w_qkv", "b_qkv") else arr
    return out


def _device_random(mesh: Mesh, rows: int, cols: int, cfg: ModelConfig, seed: int, rows_real: int | None = None):
    """Synthetic device-side init U[-1/sqrt(h), 1/sqrt(h)) in the weight layout (bench configs)."""
    lim = 1.0 / math.sqrt(cfg.h)
    gc = mesh.c
    rb, cb = rows // gc, cols // gc
    blocks = [None] * (gc * gc)
    gen = torch.Generator(device=mesh.device())
    for k in range(gc * gc):
        l, j = divmod(k, gc)
        o = mesh.flat(l % mesh.r, j)
        if not mesh.owns(o):
            continue
        gen.manual_seed(seed * 7919 + k)
        blk = mesh.persistent_empty((rb, cb), F32)
        blk.uniform_(-lim, lim, generator=gen)
        if rows_real is not None and (l + 1) * rb > rows_real:
            first_pad = max(rows_real - l * rb, 0)
            blk[first_pad:].zero_()
        blocks[k] = blk
    return _with_twin(ShardedMatrix(mesh, rows, cols, blocks, "weight"))


def run_loss_and_grads(model: MeshModel, tokens, labels, checkpointing: bool = True, cls_labels=None,
                       merge_fwd_bwd: bool = False, planned: bool = True, eager_update: bool = False,
                       lr: float = 0.0):
    """One forward + backward; returns (loss, grads, workspace, store) (model.py:414-424)."""
    ws = model.make_workspace(checkpointing=checkpointing, eager_update=eager_update, merge_fwd_bwd=merge_fwd_bwd,
                              planned=planned)
    store = CheckpointStore(model.mesh.p) if checkpointing else None
    loss, saved = model.forward(tokens, labels, ws, store=store, cls_labels=cls_labels)
    grads = model.backward(saved, ws, eager_update=eager_update, lr=lr)
    return loss, grads, ws, store
