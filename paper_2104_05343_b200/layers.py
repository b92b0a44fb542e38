"""2D transformer operators on the r x c mesh (drop-in for summagrid layers.py).

Partition (layers.py:1-21 of the reference): activations [b*s, h] are split
with token rows over mesh rows and hidden columns over mesh columns; weights
are SUMMA-partitioned; bias / LayerNorm vectors are per-column shards hosted
by row 0. The fused QKV weight is column-interleaved so column block j holds
[Q_j | K_j | V_j] for the n/c whole heads of column j; attention needs no
collective between its two SUMMA products.

B200 design choices:
  * the residual stream and every activation gradient are fp32, GEMM operands
    bf16; SUMMA partial sums accumulate in fp32;
  * bias, GELU (+ saved pre-activation), GELU' and the residual adds run in
    the GEMM epilogue (sg_gemm) instead of separate passes;
  * LayerNorm / cross-entropy move only per-row scalars across the mesh row
    (one packed (sum, sumsq) all-reduce; max + packed (sum e, x_label));
  * vectors keep a replica per mesh column, refreshed by the optimizer, so
    the reference's per-use column broadcasts (R11) disappear and their
    gradient reduces (R12) become column all-reduces.
The public functions keep the reference names, arguments and errors.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Optional

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigError, ShapeError
from .membuf import Workspace, full_storage, padded_empty
from .mesh import Mesh, MeshConfig
from .summa import (
    BF16,
    F32,
    ShardedMatrix,
    as_bf16,
    summa_ab,
    summa_abt,
    summa_abt_backward,
    summa_atb,
)


@dataclass(frozen=True)
class ModelConfig:
    """Global transformer dimensions (layers.py:45-84)."""

    b: int
    s: int
    h: int
    n: int
    v: int
    num_layers: int
    eps: float = 1e-5

    def __post_init__(self) -> None:
        if min(self.b, self.s, self.h, self.n, self.v) < 1 or self.num_layers < 0:
            raise ConfigError("model dimensions must be positive (num_layers >= 0)")
        if self.h % self.n:
            raise ConfigError(f"hidden size {self.h} not divisible by heads {self.n}")
        if self.eps <= 0:
            raise ConfigError("layer-norm eps must be > 0")

    @property
    def head_dim(self) -> int:
        return self.h // self.n

    def validate_mesh(self, q) -> None:
        """Divisibility of the 2D partition (layers.py:69-79).

        ``q`` is the square side (reference) or a Mesh / MeshConfig for r x c:
        b % r, h % c, n % c and whole heads per column shard.
        """
        r, c = _rc(q)
        for name, val, div in (("batch size b", self.b, r), ("hidden size h", self.h, c),
                               ("attention heads n", self.n, c)):
            if val % div:
                raise ConfigError(f"{name} = {val} not divisible by mesh side {div}")
        if (self.h // c) % self.head_dim:
            raise ConfigError(f"column shard h/c = {self.h // c} does not hold whole heads of size {self.head_dim}")

    def v_padded(self, q) -> int:
        """Vocabulary rounded up to a multiple of the column count (layers.py:81-84)."""
        _, c = _rc(q)
        return ((self.v + c - 1) // c) * c


def _rc(q) -> tuple[int, int]:
    if isinstance(q, int):
        return q, q
    if isinstance(q, Mesh):
        return q.r, q.c
    if isinstance(q, MeshConfig):
        return q.rows, q.cols
    raise ConfigError(f"expected a mesh side, Mesh or MeshConfig, got {type(q).__name__}")


def _qkv_perm(three_h: int, parts: int) -> np.ndarray:
    h = three_h // 3
    hp = h // parts
    return np.concatenate([np.arange(comp * h + j * hp, comp * h + (j + 1) * hp)
                           for j in range(parts) for comp in range(3)])


def interleave_qkv(w, parts: int):
    """[Q|K|V] columns -> per column-part [Q_j|K_j|V_j] (layers.py:87-102); numpy or torch."""
    idx = _qkv_perm(w.shape[-1], parts)
    return w[..., torch.as_tensor(idx, device=w.device) if isinstance(w, torch.Tensor) else idx]


def deinterleave_qkv(w, parts: int):
    """Inverse of interleave_qkv (layers.py:105-115)."""
    idx = _qkv_perm(w.shape[-1], parts)
    inv = np.empty_like(idx)
    inv[idx] = np.arange(idx.size)
    return w[..., torch.as_tensor(inv, device=w.device) if isinstance(w, torch.Tensor) else inv]


# ------------------------------------------------------------------ vectors

@dataclass
class RowHostedVector:
    """A length-W vector split into c column shards (layers.py:118-137).

    ``shards[j]`` is the fp32 shard of mesh column j. The reference hosts it
    on (0, j) and broadcasts per use; here every position of column j reads a
    replica kept in sync by the optimizer (on the dist backend each process
    holds its own column's shard; other entries are None).
    """

    shards: list

    @property
    def width(self) -> int:
        return sum(int(s.numel()) for s in self.shards if s is not None)

    def gathered(self) -> np.ndarray:
        if any(s is None for s in self.shards):
            import torch.distributed as dist

            mine = {j: s.detach().double().cpu().numpy() for j, s in enumerate(self.shards) if s is not None}
            parts = [None] * dist.get_world_size()
            dist.all_gather_object(parts, mine)
            merged = {}
            for d in parts:
                merged.update(d)
            return np.concatenate([merged[j] for j in range(len(self.shards))])
        return np.concatenate([s.detach().double().cpu().numpy() for s in self.shards])

    def for_position(self, mesh: Mesh, dev: int) -> torch.Tensor:
        return self.shards[dev % mesh.c]

    @staticmethod
    def split(vec, q, mesh: Mesh | None = None) -> "RowHostedVector":
        """Shard a host vector over the mesh columns (layers.py:132-137)."""
        _, c = _rc(mesh if mesh is not None else q)
        v = np.asarray(vec.detach().cpu() if isinstance(vec, torch.Tensor) else vec, dtype=np.float64)
        if v.size % c:
            raise ShapeError(f"vector of size {v.size} not divisible by q={c}")
        w = v.size // c
        dev = mesh.device() if mesh is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        shards = []
        for j in range(c):
            if mesh is not None and not mesh.is_local and mesh.my_flat % mesh.c != j:
                shards.append(None)
                continue
            t = padded_empty((w,), F32, dev)
            t.copy_(torch.as_tensor(v[j * w:(j + 1) * w], dtype=F32))
            shards.append(t)
        return RowHostedVector(shards)


def _vec_grad(mesh: Mesh, parts: list, tag: str) -> RowHostedVector:
    """Column all-reduce of per-position vector partials -> per-column shards (R12)."""
    mesh.allreduce_col(parts, tag=tag)
    shards = [None] * mesh.c
    for dev in mesh.local_devs:
        i, j = divmod(dev, mesh.c)
        if shards[j] is None:
            shards[j] = parts[dev]
    return RowHostedVector(shards)


# ------------------------------------------------------------------ tokens

def _token_block(tokens, row: int, r: int):
    """Flattened ids of the batch rows owned by mesh row ``row`` (layers.py:144-148)."""
    bb = tokens.shape[0] // r
    return tokens[row * bb:(row + 1) * bb].reshape(-1)


def _check_ids(ids, v: int, what: str, flag: torch.Tensor | None = None) -> None:
    """ConfigError unless every id lies in [0, v) (layers.py:164-165, 552-553).

    Host ids are checked on the host. Device ids are checked by a device kernel
    (sg_check_ids): with ``flag`` (int32 [1] on the device) the result is only
    OR-ed into it and read at the caller's next synchronisation (the step's loss
    read-back, MeshModel.check_inputs), otherwise it is read back here."""
    if isinstance(ids, torch.Tensor) and ids.is_cuda:
        flat = ids.reshape(-1)
        if flat.dtype != torch.int64 or not flat.is_contiguous():
            flat = flat.to(torch.int64).contiguous()
        own = flag is None
        if own:
            flag = torch.zeros(1, dtype=torch.int32, device=ids.device)
        K.check_ids(flat, v, flag)
        if own and int(flag.item()):
            raise ConfigError(f"{what} must lie in [0, {v})")
        return
    arr = np.asarray(ids.cpu() if isinstance(ids, torch.Tensor) else ids)
    if arr.size and (arr.min() < 0 or arr.max() >= v):
        raise ConfigError(f"{what} must lie in [0, {v})")


def _device_ids(mesh: Mesh, ids) -> list:
    """Per-position int64 device ids of the position's mesh row."""
    per_row = {}
    out = [None] * mesh.p
    for dev in mesh.local_devs:
        i = dev // mesh.c
        if i not in per_row:
            blk = _token_block(ids, i, mesh.r)
            per_row[i] = torch.as_tensor(np.ascontiguousarray(blk) if not isinstance(blk, torch.Tensor) else blk,
                                         dtype=torch.int64).to(mesh.device(dev)).contiguous()
        out[dev] = per_row[i]
    return out


# ------------------------------------------------------------------ embedding

def embedding_forward(tokens, table: ShardedMatrix, cfg: ModelConfig, ws: Workspace, out_category: str = "free",
                      tag: str = "embedding", *, ids=None) -> ShardedMatrix:
    """Token lookup in c vocabulary-block steps (layers.py:151-184).

    Step l: table block (l, j) reaches column j (R9), each position copies the
    rows of its tokens that fall in vocabulary block l.
    """
    mesh = table.mesh
    r, c = mesh.r, mesh.c
    v_pad = cfg.v_padded(mesh)
    if ids is None:  # callers passing ``ids`` validated them (MeshModel.forward)
        _check_ids(tokens, cfg.v, "token ids")
    vb, hb = v_pad // c, cfg.h // c
    bs_loc = (cfg.b // r) * cfg.s
    ids = _device_ids(mesh, tokens) if ids is None else ids
    out = [None] * mesh.p
    for dev in mesh.local_devs:
        out[dev] = ws.empty(dev, (bs_loc, hb), out_category, dtype=F32)
    pubs = None
    if not mesh.is_local and mesh.peer is not None:
        # peer memory: this position's table blocks (i + k r, j) readable by its column;
        # step l's root (l mod r, j) holds block (l, j) as its (l // r)-th block
        i, j = divmod(mesh.my_flat, c)
        pubs = [mesh.publish(f"emb{k}", table.block(i + k * r, j)) for k in range(c // r)]
        mesh.peer.barrier("col")
    for l in range(c):
        src = [None] * mesh.p
        for j in range(c):
            o = table.owner(l, j)
            if mesh.owns(o):
                src[o] = table.block(l, j)
        tab = mesh.bcast_col(l % r, src, (vb, hb), table.dtype, tag=tag,
                             views=None if pubs is None else pubs[l // r])
        for dev in mesh.local_devs:
            K.embed_fwd(ids[dev], l * vb, vb, tab[dev], out[dev])
    return ShardedMatrix(mesh, cfg.b * cfg.s, cfg.h, out)


def embedding_backward(out_grad: ShardedMatrix, tokens, table: ShardedMatrix, cfg: ModelConfig, ws: Workspace,
                       out_category: str = "free", tag: str = "embedding", *, ids=None,
                       accumulate_into: ShardedMatrix | None = None) -> ShardedMatrix:
    """Scatter-add token gradients into vocabulary rows, column-reduced to the
    block owner (layers.py:187-211); repeated ids accumulate."""
    mesh = table.mesh
    r, c = mesh.r, mesh.c
    v_pad = cfg.v_padded(mesh)
    vb, hb = v_pad // c, cfg.h // c
    ids = _device_ids(mesh, tokens) if ids is None else ids
    if accumulate_into is not None:
        res = accumulate_into
    else:
        blocks = [None] * (c * c)
        for k in range(c * c):
            o = table.owner(k // c, k % c)
            if mesh.owns(o):
                blocks[k] = ws.alloc(o, (vb, hb), out_category, dtype=F32)
        res = ShardedMatrix(mesh, v_pad, cfg.h, blocks, "weight")
    parts = [None] * mesh.p
    if not mesh.is_local:  # one staging block per position, reused by every vocabulary step
        ws.reset_all("workspace")
        for dev in mesh.local_devs:
            parts[dev] = ws.empty(dev, (vb, hb), "workspace", dtype=F32)
    for l in range(c):
        if mesh.is_local:
            # the column reduce collapses into atomics on the owner's block
            mesh.charge("reduce", "col", l % r, vb * hb, tag)
            for j in range(c):
                dst = res.block(l, j)
                for i in range(r):
                    K.embed_bwd(ids[mesh.flat(i, j)], l * vb, vb, out_grad.blocks[mesh.flat(i, j)], dst)
            continue
        for dev in mesh.local_devs:
            K.zero(full_storage(parts[dev]))
            K.embed_bwd(ids[dev], l * vb, vb, out_grad.blocks[dev], parts[dev])
        dest = [None] * mesh.p
        for j in range(c):
            o = res.owner(l, j)
            if mesh.owns(o):
                dest[o] = res.block(l, j)
        mesh.reduce_col_into(l % r, parts, dest, accumulate=True, tag=tag)
    return res


# ------------------------------------------------------------------ bias

def bias_add_forward(x: ShardedMatrix, bias: RowHostedVector, ws: Workspace, tag: str = "bias") -> ShardedMatrix:
    """x += bias shard of the position's column, in place (layers.py:218-229)."""
    mesh = x.mesh
    for dev in mesh.local_devs:
        K.bias_add(x.blocks[dev], bias.for_position(mesh, dev))
    return x


def _colsum_parts(mesh: Mesh, x: ShardedMatrix, ws: Workspace) -> list:
    parts = [None] * mesh.p
    for dev in mesh.local_devs:
        parts[dev] = ws.empty(dev, (x.block_cols,), "param_grad", dtype=F32)
        K.colsum(x.blocks[dev], parts[dev])
    return parts


def bias_add_backward(out_grad: ShardedMatrix, ws: Workspace, tag: str = "bias"):
    """(out_grad, column sums over the mesh column) (layers.py:232-246).

    When the producer of ``out_grad`` already accumulated its per-position
    column sums in its epilogue (``colsum_parts``), only the column
    all-reduce remains.
    """
    mesh = out_grad.mesh
    parts = getattr(out_grad, "colsum_parts", None)
    if parts is None:
        parts = _colsum_parts(mesh, out_grad, ws)
    else:
        out_grad.colsum_parts = None  # consumed (all-reduced in place)
    return out_grad, _vec_grad(mesh, parts, tag)


def new_colsum_parts(mesh: Mesh, ws: Workspace, width: int) -> list:
    """Zeroed per-position fp32 column-sum accumulators for a fused epilogue."""
    parts = [None] * mesh.p
    for dev in mesh.local_devs:
        parts[dev] = ws.empty(dev, (width,), "param_grad", dtype=F32)
        K.zero(parts[dev])
    return parts


# ------------------------------------------------------------------ layer norm

@dataclass
class LayerNormContext:
    """Saved state of a LayerNorm: input, per-row mean / rstd, gamma (layers.py:253-258).

    x^ is recomputed from (x, mean, rstd) in the backward kernel instead of
    being stored; ``x_hat`` materialises it for inspection.
    """

    x: ShardedMatrix
    mean: list
    rstd: list
    gamma: RowHostedVector
    h: int

    @property
    def x_hat(self) -> list:
        out = []
        for dev, xb in enumerate(self.x.blocks):
            if xb is None:
                out.append(None)
                continue
            out.append((xb.float() - self.mean[dev][:, None]) * self.rstd[dev][:, None])
        return out


def layernorm_forward(x: ShardedMatrix, gamma: RowHostedVector, beta_param: RowHostedVector, cfg: ModelConfig,
                      ws: Workspace, out_category: str = "free", tag: str = "layernorm", *,
                      out_dtype: torch.dtype = BF16):
    """Normalise over the full hidden size with one packed row all-reduce (layers.py:261-307)."""
    mesh = x.mesh
    rows, cols = x.block_rows, x.block_cols
    stats = [None] * mesh.p
    if mesh.c > 1:
        for dev in mesh.local_devs:
            stats[dev] = ws.empty(dev, (rows, 2), "free", dtype=F32, pad=False)
            K.ln_stats(x.blocks[dev], stats[dev])
        mesh.allreduce_row(stats, tag=tag)
    y, mean, rstd = [None] * mesh.p, [None] * mesh.p, [None] * mesh.p
    for dev in mesh.local_devs:
        y[dev] = ws.empty(dev, (rows, cols), out_category, dtype=out_dtype)
        mean[dev] = ws.empty(dev, (rows,), "free", dtype=F32)
        rstd[dev] = ws.empty(dev, (rows,), "free", dtype=F32)
        K.ln_fwd(x.blocks[dev], stats[dev], cfg.h, cfg.eps, gamma.for_position(mesh, dev),
                 beta_param.for_position(mesh, dev), y[dev], mean[dev], rstd[dev])
    return (ShardedMatrix(mesh, x.global_rows, x.global_cols, y),
            LayerNormContext(x=x, mean=mean, rstd=rstd, gamma=gamma, h=cfg.h))


def layernorm_backward(out_grad: ShardedMatrix, ctx: LayerNormContext, cfg: ModelConfig, ws: Workspace,
                       out_category: str = "free", tag: str = "layernorm", *, resid: ShardedMatrix | None = None,
                       want_bf16: bool = False, want_colsum: bool = False):
    """dx = rstd (g - mean_h g - x^ mean_h(x^ g)), g = dy gamma; the two row sums in
    one packed all-reduce; (dgamma, dbeta) column-all-reduced (layers.py:310-351).

    ``resid`` adds a residual-stream gradient in the same pass; with
    ``want_bf16`` the result also carries a bf16 twin for the next GEMMs and
    with ``want_colsum`` its column sums (the upstream bias gradient).
    """
    mesh = out_grad.mesh
    rows, cols = out_grad.block_rows, out_grad.block_cols
    stats = getattr(out_grad, "ln_stats", None)  # accumulated by the producing GEMM (summa_abt ln_ctx)
    if stats is None:
        stats = [None] * mesh.p
        for dev in mesh.local_devs:
            stats[dev] = ws.empty(dev, (rows, 2), "free", dtype=F32, pad=False)
            K.ln_bwd_stats(out_grad.blocks[dev], ctx.x.blocks[dev], ctx.mean[dev], ctx.rstd[dev],
                           ctx.gamma.for_position(mesh, dev), stats[dev])
    if mesh.c > 1:
        mesh.allreduce_row(stats, tag=tag)
    dx, dx16, gb = [None] * mesh.p, [None] * mesh.p, [None] * mesh.p
    dsum = new_colsum_parts(mesh, ws, cols) if want_colsum else [None] * mesh.p
    for dev in mesh.local_devs:
        dx[dev] = ws.empty(dev, (rows, cols), out_category, dtype=F32)
        if want_bf16:
            dx16[dev] = ws.empty(dev, (rows, cols), "free", dtype=BF16)
        gb[dev] = ws.empty(dev, (2, cols), "param_grad", dtype=F32, pad=False)
        K.zero(gb[dev])
        K.ln_bwd(out_grad.blocks[dev], ctx.x.blocks[dev], ctx.mean[dev], ctx.rstd[dev],
                 ctx.gamma.for_position(mesh, dev), stats[dev], cfg.h,
                 None if resid is None else resid.blocks[dev], dx[dev], dx16[dev], gb[dev][0], gb[dev][1],
                 dsum[dev])
    flat = [None if g is None else g.reshape(-1) for g in gb]
    mesh.allreduce_col(flat, tag=tag)
    g_sh, b_sh = [None] * mesh.c, [None] * mesh.c
    for dev in mesh.local_devs:
        j = dev % mesh.c
        if g_sh[j] is None:
            g_sh[j], b_sh[j] = flat[dev][:cols], flat[dev][cols:2 * cols]
    out = ShardedMatrix(mesh, out_grad.global_rows, out_grad.global_cols, dx)
    if want_bf16:
        out.bf16_twin = ShardedMatrix(mesh, out_grad.global_rows, out_grad.global_cols, dx16)
    if want_colsum:
        out.colsum_parts = dsum
    return out, RowHostedVector(g_sh), RowHostedVector(b_sh)


# ------------------------------------------------------------------ attention

@dataclass
class AttentionContext:
    """Saved attention state (layers.py:358-365): input, QKV block, context.

    On the flash path the per-row log-sum-exp replaces P; ``probs`` is then
    rebuilt on demand (the backward never needs it).
    """

    x_in: ShardedMatrix
    qkv: ShardedMatrix
    saved_probs: list
    ctx_mat: ShardedMatrix
    cfg: ModelConfig
    lse: list | None = None

    @property
    def probs(self) -> list:
        mesh = self.qkv.mesh
        for dev in mesh.local_devs:
            if self.saved_probs[dev] is None:
                self.saved_probs[dev] = _probs(self.cfg, mesh, self.qkv.blocks[dev], dev)
        return self.saved_probs

    def _heads(self, part: int) -> list:
        mesh = self.qkv.mesh
        b_loc, n_loc, d = self.cfg.b // mesh.r, self.cfg.n // mesh.c, self.cfg.head_dim
        hb = self.cfg.h // mesh.c
        out = []
        for blk in self.qkv.blocks:
            out.append(None if blk is None else _heads_view(blk[:, part * hb:(part + 1) * hb], b_loc, self.cfg.s,
                                                            n_loc, d))
        return out

    @property
    def q_heads(self) -> list:
        return self._heads(0)

    @property
    def k_heads(self) -> list:
        return self._heads(1)

    @property
    def v_heads(self) -> list:
        return self._heads(2)


def _heads_view(blk: torch.Tensor, b_loc: int, s: int, n_loc: int, d: int) -> torch.Tensor:
    """[b*s, n*d] block (any row pitch) -> strided [b, n, s, d] view, no copy (layers.py:368-377)."""
    ld = blk.stride(0)
    return torch.as_strided(blk, (b_loc, n_loc, s, d), (s * ld, d, ld, 1))


# The softmax-backward epilogue reads P per 32-column chunk and is latency-bound on
# that input; the unfused dP product + row kernel is faster until attention moves to
# a flash-style kernel.
FUSED_SOFTMAX_BWD = False


def fused_softmax_ok(cfg: ModelConfig) -> bool:
    """The row-softmax GEMM epilogues hold a whole score row in TMEM (s <= 512)
    and need TMA-aligned head slices."""
    return cfg.s <= 512 and cfg.s % 8 == 0 and cfg.head_dim % 8 == 0


def flash_ok(cfg: ModelConfig) -> bool:
    """The tcgen05 flash forward (sg_attn.cu) covers head_dim 64 and 128 at any sequence length."""
    return FLASH_ATTENTION and cfg.head_dim in (64, 128)


def flash_bwd_ok(cfg: ModelConfig) -> bool:
    """The flash backward covers head_dim 64 and 128; otherwise P is rebuilt from Q, K (AttentionContext.probs)."""
    return FLASH_ATTENTION and cfg.head_dim in (64, 128)


FLASH_ATTENTION = True


def _probs(cfg: ModelConfig, mesh: Mesh, qkv_blk, dev):
    """P = softmax(Q K^T / sqrt(d)) as bf16 [b, n, s, s] (the reference's saved ``probs``)."""
    return _probs_core(cfg, cfg.b // mesh.r, cfg.n // mesh.c, qkv_blk, mesh.device(dev))


def _probs_core(cfg: ModelConfig, b_loc: int, n_loc: int, qkv_blk, device):
    d, s = cfg.head_dim, cfg.s
    hb = n_loc * d
    q = _heads_view(qkv_blk[:, :hb], b_loc, s, n_loc, d)
    k = _heads_view(qkv_blk[:, hb:2 * hb], b_loc, s, n_loc, d)
    probs = padded_empty((b_loc, n_loc, s, s), BF16, device)
    if fused_softmax_ok(cfg):
        # P straight out of TMEM: no fp32 score matrix in HBM
        K.gemm(q, k.transpose(-1, -2), probs, alpha=1.0 / math.sqrt(d), mode=K.EPI_SOFTMAX)
    else:
        scores = padded_empty((b_loc, n_loc, s, s), F32, device)
        K.gemm(q, k.transpose(-1, -2), scores, alpha=1.0 / math.sqrt(d))
        K.softmax_rows(_rows_view(scores), _rows_view(probs))
    return probs


def _local_attention(cfg: ModelConfig, mesh: Mesh, qkv_blk, ctx_blk, ws, dev):
    """Per-position multi-head attention on one block; returns (probs | None, lse | None)."""
    return attention_core_forward(cfg, cfg.b // mesh.r, cfg.n // mesh.c, qkv_blk, ctx_blk, ws, dev, mesh.device(dev))


def attention_core_forward(cfg: ModelConfig, b_loc: int, n_loc: int, qkv_blk, ctx_blk, ws, dev, device):
    """softmax(Q K^T / sqrt(d)) V for the b_loc sequences x n_loc heads of one
    position's [b_loc*s, 3*n_loc*d] QKV block (layers.py:404-416); returns
    (probs | None, lse | None)."""
    d, s = cfg.head_dim, cfg.s
    hb = n_loc * d
    if flash_ok(cfg):
        lse = ws.empty(dev, (b_loc, n_loc, s), "forward", dtype=F32, pad=False)
        K.flash_attn_fwd(qkv_blk, b_loc, s, n_loc, d, ctx_blk, lse)
        return None, lse
    probs = _probs_core(cfg, b_loc, n_loc, qkv_blk, device)
    v = _heads_view(qkv_blk[:, 2 * hb:], b_loc, s, n_loc, d)
    K.gemm(probs, v, _heads_view(ctx_blk, b_loc, s, n_loc, d))
    return probs, None


def _rows_view(t: torch.Tensor) -> torch.Tensor:
    """[..., s] padded tensor -> 2-D [rows, s] view with the padded pitch."""
    return torch.as_strided(t, (t.numel() // t.shape[-1], t.shape[-1]), (t.stride(-2), 1))


def attention_forward(x: ShardedMatrix, w_qkv: ShardedMatrix, b_qkv: RowHostedVector, w_dense: ShardedMatrix,
                      b_dense: RowHostedVector, cfg: ModelConfig, ws: Workspace, *,
                      resid: ShardedMatrix | None = None):
    """QKV product, per-position multi-head attention, dense product (layers.py:380-421).

    No collective between the two SUMMA products; biases (and the optional
    residual) are added in the GEMM epilogues.
    """
    mesh = x.mesh
    cfg.validate_mesh(mesh)
    hb = cfg.h // mesh.c
    bs_loc = (cfg.b // mesh.r) * cfg.s
    qkv = _tagged("qkv", summa_ab, x, w_qkv, ws, out_category="forward", tag="summa", out_dtype=BF16,
                   bias=[None if d is None else b_qkv.for_position(mesh, d) for d in _all(mesh)])
    ctx_blocks, probs, lse = [None] * mesh.p, [None] * mesh.p, [None] * mesh.p
    mac_per_dev = (cfg.b // mesh.r) * (cfg.n // mesh.c) * cfg.s * cfg.s * cfg.head_dim
    mesh.add_macs_all(2 * mac_per_dev)  # QK^T, PV (layers.py:414)
    for dev in mesh.local_devs:
        ctx_blocks[dev] = ws.empty(dev, (bs_loc, hb), "free", dtype=BF16)
        probs[dev], lse[dev] = _local_attention(cfg, mesh, qkv.blocks[dev], ctx_blocks[dev], ws, dev)
    ctx_mat = ShardedMatrix(mesh, cfg.b * cfg.s, cfg.h, ctx_blocks)
    out = _tagged("dense", summa_ab, ctx_mat, w_dense, ws, out_category="forward", tag="summa", out_dtype=F32,
                   bias=[None if d is None else b_dense.for_position(mesh, d) for d in _all(mesh)], resid=resid)
    return out, AttentionContext(x_in=x, qkv=qkv, saved_probs=probs, ctx_mat=ctx_mat, cfg=cfg,
                                 lse=lse if flash_ok(cfg) else None)


def attention_core_backward(cfg: ModelConfig, b_loc: int, n_loc: int, qkv_blk, ctx_blk, dctx_blk, lse, probs_fn, ws,
                            dev, device, bq_part):
    """dQKV [b_loc*s, 3*n_loc*d] (bf16) of one position's attention core from dO = dctx
    (layers.py:444-459); ``bq_part`` (fp32 [3*n_loc*d]) accumulates its column sums
    (the b_qkv gradient). Flash path from the saved lse, otherwise through P
    (``probs_fn()`` returns it, rebuilt if it was not kept)."""
    d, s = cfg.head_dim, cfg.s
    hb = n_loc * d
    bs_loc = b_loc * s
    scale = 1.0 / math.sqrt(d)
    q = _heads_view(qkv_blk[:, :hb], b_loc, s, n_loc, d)
    k = _heads_view(qkv_blk[:, hb:2 * hb], b_loc, s, n_loc, d)
    v = _heads_view(qkv_blk[:, 2 * hb:], b_loc, s, n_loc, d)
    dq_blk = ws.empty(dev, (bs_loc, 3 * hb), "free", dtype=BF16)
    if lse is not None and flash_bwd_ok(cfg):
        # flash backward: P rebuilt per tile from lse, never in HBM; D = rowsum(dO O)
        drow = ws.empty(dev, (b_loc, n_loc, s), "free", dtype=F32, pad=False)
        K.attn_rowdot(dctx_blk, ctx_blk, n_loc, d, s, drow)
        dq_acc = ws.alloc(dev, (bs_loc, hb), "free", dtype=F32)
        fused = hb % 256 == 0
        # the K / V parts of the b_qkv gradient summed from the staged dK / dV tiles
        K.flash_attn_bwd(qkv_blk, dctx_blk, lse, drow, b_loc, s, n_loc, d, dq_acc, dq_blk,
                         kv_colsum=bq_part[hb:] if fused else None)
        if fused:  # dQ to bf16 and its b_qkv gradient part in one pass
            K.qkv_grad_finish(dq_acc, dq_blk, hb, bq_part, q_only=True)
        else:
            K.epilogue(dq_acc, dq_blk[:, :hb])
            K.colsum(dq_blk, bq_part, accumulate=True)
        return dq_blk
    dheads = _heads_view(dctx_blk, b_loc, s, n_loc, d)
    p_mat = probs_fn()
    cs = [bq_part[i * hb:(i + 1) * hb].view(1, n_loc, d) for i in range(3)]
    ds = padded_empty((b_loc, n_loc, s, s), BF16, device)
    if fused_softmax_ok(cfg) and FUSED_SOFTMAX_BWD:
        # dS = P (dP - D) / sqrt(d) straight out of the dP = dO V^T accumulator, with
        # D = rowsum(dP P) = rowsum(dO O) computed from the saved context
        drow = padded_empty((b_loc, n_loc, s), F32, device)
        K.attn_rowdot(dctx_blk, ctx_blk, n_loc, d, s, drow)
        K.gemm(dheads, v.transpose(-1, -2), ds, alpha=scale, mode=K.EPI_SOFTMAX_BWD, aux=p_mat, rowvec=drow)
    else:
        dp = padded_empty((b_loc, n_loc, s, s), F32, device)
        K.gemm(dheads, v.transpose(-1, -2), dp)                              # dP = dO V^T
        K.softmax_bwd(_rows_view(dp), _rows_view(p_mat), scale, _rows_view(ds))
    K.gemm(p_mat.transpose(-1, -2), dheads, _heads_view(dq_blk[:, 2 * hb:], b_loc, s, n_loc, d),
           colsum=cs[2])                                                     # dV = P^T dO
    K.gemm(ds, k, _heads_view(dq_blk[:, :hb], b_loc, s, n_loc, d), colsum=cs[0])          # dQ = dS K
    K.gemm(ds.transpose(-1, -2), q, _heads_view(dq_blk[:, hb:2 * hb], b_loc, s, n_loc, d),
           colsum=cs[1])                                                     # dK = dS^T Q
    return dq_blk


def _tagged(name: str, fn, *args, **kw):
    """Run a SUMMA product with its GEMM launches labelled ``name`` (bench roofline list)."""
    with K.tagged(name):
        return fn(*args, **kw)


def _all(mesh: Mesh) -> list:
    return [d if mesh.owns(d) else None for d in range(mesh.p)]


def _bf16_of(x: ShardedMatrix, ws: Workspace) -> ShardedMatrix:
    twin = getattr(x, "bf16_twin", None)
    return twin if twin is not None else as_bf16(x)


def _weight_grad(a: ShardedMatrix, b: ShardedMatrix, w: ShardedMatrix, ws: Workspace, lr):
    """dW = a^T b, or with ``lr`` (eager SGD; local mesh, or dist mesh with peer memory)
    w -= lr a^T b in place by the product's (remote) reduce-add epilogue (returns None:
    no gradient is materialised)."""
    if lr is not None and (a.mesh.is_local or a.mesh.peer is not None):
        summa_atb(a, b, ws, accumulate_into=w, alpha=-lr)
        return None
    return summa_atb(a, b, ws, out_category="param_grad")


def attention_backward(out_grad: ShardedMatrix, ctx: AttentionContext, w_qkv: ShardedMatrix,
                       w_dense: ShardedMatrix, cfg: ModelConfig, ws: Workspace, ln_ctx=None, lr=None):
    """(dx, dW_qkv, db_qkv, dW_dense, db_dense) (layers.py:424-465); ``ln_ctx`` is
    the LayerNorm whose backward consumes dx (its statistics fused into dx's GEMM);
    ``lr``: weights updated in place by their gradient products (dW entries None)."""
    mesh = out_grad.mesh
    b_loc, n_loc = cfg.b // mesh.r, cfg.n // mesh.c
    hb = cfg.h // mesh.c
    dy16 = _bf16_of(out_grad, ws)
    _, b_dense_grad = bias_add_backward(out_grad, ws)
    dctx = _tagged("dctx", summa_abt, dy16, w_dense, ws, out_category="backward", out_dtype=BF16)
    w_dense_grad = _tagged("dw_dense", _weight_grad, ctx.ctx_mat, dy16, w_dense, ws, lr)
    bq_parts = new_colsum_parts(mesh, ws, 3 * hb)  # b_qkv gradient fused into dQ / dK / dV epilogues
    mesh.add_macs_all(4 * b_loc * n_loc * cfg.s * cfg.s * cfg.head_dim)  # dP, dV, dQ, dK (layers.py:457)
    dqkv_blocks = [None] * mesh.p
    for dev in mesh.local_devs:
        dqkv_blocks[dev] = attention_core_backward(
            cfg, b_loc, n_loc, ctx.qkv.blocks[dev], ctx.ctx_mat.blocks[dev], dctx.blocks[dev],
            None if ctx.lse is None else ctx.lse[dev], lambda dev=dev: ctx.probs[dev], ws, dev, mesh.device(dev),
            bq_parts[dev])
    dqkv = ShardedMatrix(mesh, cfg.b * cfg.s, 3 * cfg.h, dqkv_blocks)
    dqkv.colsum_parts = bq_parts
    _, b_qkv_grad = bias_add_backward(dqkv, ws)
    x_grad = _tagged("dx_qkv", summa_abt, dqkv, w_qkv, ws, out_category="backward", out_dtype=F32, ln_ctx=ln_ctx)
    w_qkv_grad = _tagged("dw_qkv", _weight_grad, ctx.x_in, dqkv, w_qkv, ws, lr)
    return x_grad, w_qkv_grad, b_qkv_grad, w_dense_grad, b_dense_grad


# ------------------------------------------------------------------ MLP

@dataclass
class MlpContext:
    """x, the h->4h pre-activation (GELU' input) and gelu(mid) (layers.py:472-476)."""

    x_in: ShardedMatrix
    mid: ShardedMatrix
    act: ShardedMatrix


def mlp_forward(x: ShardedMatrix, w1: ShardedMatrix, b1: RowHostedVector, w2: ShardedMatrix,
                b2: RowHostedVector, cfg: ModelConfig, ws: Workspace, *, resid: ShardedMatrix | None = None):
    """h->4h product (+b1, GELU fused, pre-activation saved), 4h->h product (+b2) (layers.py:479-491)."""
    mesh = x.mesh
    rows, cols4 = x.block_rows, 4 * cfg.h // mesh.c
    mid_blocks = [None] * mesh.p
    for dev in mesh.local_devs:
        mid_blocks[dev] = ws.empty(dev, (rows, cols4), "forward", dtype=BF16)
    mid = ShardedMatrix(mesh, x.global_rows, 4 * cfg.h, mid_blocks)
    act = _tagged("fc1", summa_ab, x, w1, ws, out_category="free", tag="summa", out_dtype=BF16,
                   bias=[None if d is None else b1.for_position(mesh, d) for d in _all(mesh)], act=K.ACT_GELU,
                   aux=mid)
    out = _tagged("fc2", summa_ab, act, w2, ws, out_category="forward", tag="summa", out_dtype=F32,
                   bias=[None if d is None else b2.for_position(mesh, d) for d in _all(mesh)], resid=resid)
    return out, MlpContext(x_in=x, mid=mid, act=act)


def mlp_backward(out_grad: ShardedMatrix, ctx: MlpContext, w1: ShardedMatrix, w2: ShardedMatrix,
                 cfg: ModelConfig, ws: Workspace, ln_ctx=None, lr=None):
    """(dx, dW1, db1, dW2, db2) with GELU' fused into the dAct product (layers.py:494-508);
    ``ln_ctx``, ``lr`` as in attention_backward."""
    mesh = out_grad.mesh
    dy16 = _bf16_of(out_grad, ws)
    _, b2_grad = bias_add_backward(out_grad, ws)
    b1_parts = new_colsum_parts(mesh, ws, ctx.mid.block_cols)
    # GELU' (from the saved pre-activation, TMA-loaded per output tile) and the b1
    # gradient column sums fused into the dAct product's epilogue (layers.py:502-504)
    dmid = _tagged("dact", summa_abt, dy16, w2, ws, out_category="backward", out_dtype=BF16, act=K.ACT_DGELU, aux=ctx.mid,
                     colsum=b1_parts)
    dmid.colsum_parts = b1_parts
    w2_grad = _tagged("dw2", _weight_grad, ctx.act, dy16, w2, ws, lr)
    _, b1_grad = bias_add_backward(dmid, ws)
    x_grad = _tagged("dx_fc1", summa_abt, dmid, w1, ws, out_category="backward", out_dtype=F32, ln_ctx=ln_ctx)
    w1_grad = _tagged("dw1", _weight_grad, ctx.x_in, dmid, w1, ws, lr)
    return x_grad, w1_grad, b1_grad, w2_grad, b2_grad


# ------------------------------------------------------------------ lm head + cross entropy

def lm_head_logits(x: ShardedMatrix, table: ShardedMatrix, ws: Workspace, out_category: str = "free",
                   tag: str = "lmhead", *, out_dtype: torch.dtype = F32) -> ShardedMatrix:
    """Vocabulary logits x table^T on the embedding's partition (layers.py:515-518)."""
    return summa_abt(x, table, ws, out_category=out_category, tag=tag, out_dtype=out_dtype)


def lm_head_backward(logits_grad: ShardedMatrix, x: ShardedMatrix, table: ShardedMatrix, ws: Workspace,
                     x_out_category: str = "free", w_out_category: str = "free", tag: str = "lmhead"):
    """(dx, dtable) of the tied head (layers.py:521-527)."""
    return summa_abt_backward(logits_grad, x, table, ws, a_out_category=x_out_category,
                              b_out_category=w_out_category, tag=tag)


@dataclass
class CrossEntropyContext:
    """Row statistics of the vocab-parallel softmax (layers.py:530-536).

    Instead of materialising the softmax shards, the context keeps the logits,
    the row max and the row sum; the backward recomputes softmax - onehot in
    one pass. ``softmax`` materialises them for inspection.
    """

    logits: ShardedMatrix
    labels: list
    gmax: list
    packed: list
    loss_rows: list
    n_real: list
    tokens_total: int
    v: int

    @property
    def loss_per_token(self) -> list:
        return self.loss_rows

    @property
    def softmax(self) -> list:
        out = []
        for dev, lg in enumerate(self.logits.blocks):
            if lg is None:
                out.append(None)
                continue
            sm = torch.exp(lg.float() - self.gmax[dev][:, None]) / self.packed[dev][:, 0:1]
            sm[:, self.n_real[dev]:] = 0.0
            out.append(sm)
        return out


def cross_entropy_forward(logits: ShardedMatrix, labels, cfg: ModelConfig, ws: Workspace, tag: str = "loss", *,
                          label_ids=None, return_tensor: bool = False):
    """Mean token cross entropy over b*s (layers.py:539-608).

    Row max all-reduce, then one packed (sum e^{x-max}, x_label) all-reduce and
    a column all-reduce of the per-position loss sums. Padded vocabulary
    columns are masked out.
    """
    mesh = logits.mesh
    r, c = mesh.r, mesh.c
    v_pad = cfg.v_padded(mesh)
    vb = v_pad // c
    if label_ids is None:  # callers passing ``label_ids`` validated them (MeshModel.forward)
        _check_ids(labels, cfg.v, "labels")
    labs = _device_ids(mesh, labels) if label_ids is None else label_ids
    rows = logits.block_rows
    lmax, gmax, packed, loss_rows, part, n_real = ([None] * mesh.p for _ in range(6))
    for dev in mesh.local_devs:
        j = dev % c
        n_real[dev] = min(max(cfg.v - j * vb, 0), vb)
        lmax[dev] = ws.empty(dev, (rows,), "free", dtype=F32)
        gmax[dev] = ws.empty(dev, (rows,), "free", dtype=F32)
        packed[dev] = ws.empty(dev, (rows, 2), "free", dtype=F32, pad=False)
        K.xent_local(logits.blocks[dev], n_real[dev], labs[dev], j * vb, lmax[dev], gmax[dev], packed[dev])
    if c > 1:
        mesh.allreduce_row(gmax, op="max", tag=tag)
        for dev in mesh.local_devs:
            K.xent_rescale(lmax[dev], gmax[dev], packed[dev])
        mesh.allreduce_row(packed, tag=tag)
    for dev in mesh.local_devs:
        loss_rows[dev] = ws.empty(dev, (rows,), "free", dtype=F32)
        part[dev] = ws.empty(dev, (1,), "free", dtype=F32)
        K.xent_loss(gmax[dev], packed[dev], loss_rows[dev], part[dev])
    mesh.allreduce_col(part, tag=tag)
    tokens_total = cfg.b * cfg.s
    ctx = CrossEntropyContext(logits=logits, labels=labs, gmax=gmax, packed=packed, loss_rows=loss_rows,
                              n_real=n_real, tokens_total=tokens_total, v=cfg.v)
    first = mesh.local_devs[0]
    total = part[first] / tokens_total
    if return_tensor:
        return total, ctx
    return float(total.item()), ctx


def cross_entropy_backward(ctx: CrossEntropyContext, mesh: Mesh, ws: Workspace, upstream: float = 1.0,
                           out_category: str = "free", *, out_dtype: torch.dtype = F32, in_place: bool = False):
    """Per-position dlogits = (softmax - onehot) * upstream / (b*s) (layers.py:611-624).

    Returns the list of per-position blocks (the reference returns a list).
    ``in_place`` overwrites the logits buffer (same dtype) to save HBM.
    """
    scale = upstream / ctx.tokens_total
    vb = ctx.logits.block_cols
    out = [None] * mesh.p
    for dev in mesh.local_devs:
        lg = ctx.logits.blocks[dev]
        g = lg if in_place else ws.empty(dev, tuple(lg.shape), out_category, dtype=out_dtype)
        K.xent_bwd(lg, ctx.n_real[dev], ctx.labels[dev], (dev % mesh.c) * vb, ctx.gmax[dev], ctx.packed[dev],
                   scale, g)
        out[dev] = g
    return out


# ------------------------------------------------------------------ transformer layer

@dataclass
class LayerParams:
    w_qkv: ShardedMatrix
    b_qkv: RowHostedVector
    w_dense: ShardedMatrix
    b_dense: RowHostedVector
    w1: ShardedMatrix
    b1: RowHostedVector
    w2: ShardedMatrix
    b2: RowHostedVector
    ln1_gamma: RowHostedVector
    ln1_beta: RowHostedVector
    ln2_gamma: RowHostedVector
    ln2_beta: RowHostedVector


@dataclass
class LayerGrads:
    w_qkv: ShardedMatrix
    b_qkv: RowHostedVector
    w_dense: ShardedMatrix
    b_dense: RowHostedVector
    w1: ShardedMatrix
    b1: RowHostedVector
    w2: ShardedMatrix
    b2: RowHostedVector
    ln1_gamma: RowHostedVector
    ln1_beta: RowHostedVector
    ln2_gamma: RowHostedVector
    ln2_beta: RowHostedVector


@dataclass
class LayerSaved:
    x_in: ShardedMatrix
    ln1: LayerNormContext
    attn: AttentionContext
    y1: ShardedMatrix
    ln2: LayerNormContext
    mlp: MlpContext
    out: ShardedMatrix


_MATS = ("w_qkv", "w_dense", "w1", "w2")
_VECS = ("b_qkv", "b_dense", "b1", "b2", "ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta")


class TransformerLayer:
    """Pre-norm layer y1 = x + Attn(LN1 x); out = y1 + MLP(LN2 y1) (layers.py:674-772).

    Residual adds are fused into the dense / fc2 GEMM epilogues; the backward
    fuses the residual-gradient adds into the two LayerNorm backward passes.
    """

    fused_sgd = True  # backward(lr=...) updates the weight matrices inside their dW products

    def __init__(self, mesh: Mesh, cfg: ModelConfig, params: LayerParams, skip_dead_recompute: bool = False) -> None:
        self.mesh = mesh
        self.cfg = cfg
        self.params = params
        self.skip_dead_recompute = skip_dead_recompute
        self._recompute_mode = False
        self._last_was_skip = False

    def recompute_forward(self, x: ShardedMatrix, ws: Workspace):
        self._recompute_mode = True
        try:
            return self.forward(x, ws)
        finally:
            self._recompute_mode = False

    def forward(self, x: ShardedMatrix, ws: Workspace):
        p, cfg = self.params, self.cfg
        self._last_was_skip = self._recompute_mode and self.skip_dead_recompute
        a1, ln1 = layernorm_forward(x, p.ln1_gamma, p.ln1_beta, cfg, ws)
        y1, attn = attention_forward(a1, p.w_qkv, p.b_qkv, p.w_dense, p.b_dense, cfg, ws, resid=x)
        a2, ln2 = layernorm_forward(y1, p.ln2_gamma, p.ln2_beta, cfg, ws)
        if self._last_was_skip:
            mesh = self.mesh
            mid_blocks = [None] * mesh.p
            for dev in mesh.local_devs:
                mid_blocks[dev] = ws.empty(dev, (a2.block_rows, 4 * cfg.h // mesh.c), "forward", dtype=BF16)
            mid = ShardedMatrix(mesh, a2.global_rows, 4 * cfg.h, mid_blocks)
            act = _tagged("fc1", summa_ab, a2, p.w1, ws, out_category="free", out_dtype=BF16,
                           bias=[None if d is None else p.b1.for_position(mesh, d) for d in _all(mesh)],
                           act=K.ACT_GELU, aux=mid)
            mlp = MlpContext(x_in=a2, mid=mid, act=act)
            out = y1  # the 4h->h output feeds only the (checkpointed) next layer
        else:
            out, mlp = mlp_forward(a2, p.w1, p.b1, p.w2, p.b2, cfg, ws, resid=y1)
        return out, LayerSaved(x_in=x, ln1=ln1, attn=attn, y1=y1, ln2=ln2, mlp=mlp, out=out)

    def backward(self, out_grad: ShardedMatrix, saved: LayerSaved, ws: Workspace, lr=None):
        """Layer gradients; with ``lr`` (eager SGD) the four weight matrices are updated in
        place by their gradient products and their LayerGrads entries are None."""
        cfg, mesh, p = self.cfg, self.mesh, self.params
        bsh_p = (cfg.b * cfg.s // mesh.r) * (cfg.h // mesh.c)
        for dev in mesh.local_devs:
            ws.release_forward(dev, (4 if self._last_was_skip else 5) * bsh_p)
        da2, w1_g, b1_g, w2_g, b2_g = mlp_backward(out_grad, saved.mlp, p.w1, p.w2, cfg, ws, ln_ctx=saved.ln2,
                                                   lr=lr)
        dy1, ln2_g, ln2_b = layernorm_backward(da2, saved.ln2, cfg, ws, resid=out_grad, want_bf16=True,
                                               want_colsum=True)
        da1, wqkv_g, bqkv_g, wd_g, bd_g = attention_backward(dy1, saved.attn, p.w_qkv, p.w_dense, cfg, ws,
                                                             ln_ctx=saved.ln1, lr=lr)
        dx, ln1_g, ln1_b = layernorm_backward(da1, saved.ln1, cfg, ws, resid=dy1, want_bf16=True,
                                              want_colsum=True)
        return dx, LayerGrads(w_qkv=wqkv_g, b_qkv=bqkv_g, w_dense=wd_g, b_dense=bd_g, w1=w1_g, b1=b1_g, w2=w2_g,
                              b2=b2_g, ln1_gamma=ln1_g, ln1_beta=ln1_b, ln2_gamma=ln2_g, ln2_beta=ln2_b)

    def apply_sgd(self, grads: LayerGrads, lr: float) -> None:
        """w -= lr g on the fp32 masters, refreshing the bf16 GEMM copies (layers.py:761-772);
        all twelve parameters in one multi-tensor launch."""
        triples = []
        for name in _MATS:
            triples += _sgd_triples_matrix(getattr(self.params, name), getattr(grads, name))
        for name in _VECS:
            triples += _sgd_triples_vector(getattr(self.params, name), getattr(grads, name))
        K.sgd_multi(triples, lr)


def _sgd_triples_matrix(w: ShardedMatrix, g: ShardedMatrix | None) -> list:
    """(w, bf16 twin, g) per block; g None: w already updated, refresh the twin only."""
    twin = getattr(w, "bf16_twin", None)
    return [(blk, None if twin is None else twin.blocks[k], None if g is None else g.blocks[k])
            for k, blk in enumerate(w.blocks) if blk is not None]


def _sgd_triples_vector(v: RowHostedVector, g: RowHostedVector) -> list:
    return [(s, None, g.shards[j]) for j, s in enumerate(v.shards) if s is not None]


def sgd_matrix(w: ShardedMatrix, g: ShardedMatrix, lr: float) -> None:
    K.sgd_multi(_sgd_triples_matrix(w, g), lr)


def sgd_vector(v: RowHostedVector, g: RowHostedVector, lr: float) -> None:
    K.sgd_multi(_sgd_triples_vector(v, g), lr)
