"""SUMMA block products C = AB, C = AB^T, C = A^T B on the r x c mesh.

Drop-in for summagrid summa.py:30-191 (same names, arguments, errors and
block layout for square meshes). Each SUMMA step is: panel broadcasts over
the mesh row / column, then the local product on the tcgen05 tensor cores
(libsg ``sg_gemm``) accumulating in fp32 in step order l = 0..c-1; the AB^T /
A^T B forms reduce partial products over the row / column in group-position
order. On the single-GPU (local) mesh the reduce is fused into the
accumulating GEMM: the destination block is built as an ordered chain of
GEMMs with C = D, no partial buffers and no separate reduction pass.

Layouts (the r x c generalisation):
  * "act"    — r x c block grid, block (i, j) on position (i, j): activations,
               rows (tokens) split over mesh rows, columns over mesh columns.
  * "weight" — c x c block grid, block (l, j) on position (l mod r, j).
For r == c both are the reference's q x q layout (summa.py:30-56).
  summa_ab : act x weight -> act      summa_abt: act x weight -> act
  summa_atb: act x act    -> weight
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import kernels as K
from .errors import ConfigError, ShapeError
from .membuf import copy_block, full_storage, padded_empty
from .mesh import Mesh, check_same_mesh

BF16 = torch.bfloat16
F32 = torch.float32


@dataclass
class ShardedMatrix:
    """A global matrix split into blocks over the mesh.

    ``blocks`` is indexed by block-grid position (row * grid_cols + col); for
    the "act" layout that is the owning position's flat rank, as in the
    reference. Entries of blocks owned by other processes are None.
    """

    mesh: Mesh
    global_rows: int
    global_cols: int
    blocks: list
    layout: str = "act"

    @property
    def grid(self) -> tuple[int, int]:
        return (self.mesh.r, self.mesh.c) if self.layout == "act" else (self.mesh.c, self.mesh.c)

    @property
    def block_rows(self) -> int:
        return self.global_rows // self.grid[0]

    @property
    def block_cols(self) -> int:
        return self.global_cols // self.grid[1]

    def block(self, row: int, col: int):
        return self.blocks[row * self.grid[1] + col]

    def owner(self, row: int, col: int) -> int:
        if self.layout == "act":
            return self.mesh.flat(row, col)
        return self.mesh.flat(row % self.mesh.r, col)

    def owned_indices(self) -> list[int]:
        gc = self.grid[1]
        return [k for k in range(len(self.blocks)) if self.mesh.owns(self.owner(k // gc, k % gc))]

    @property
    def dtype(self):
        for b in self.blocks:
            if b is not None:
                return b.dtype
        return None

    def copy(self) -> "ShardedMatrix":
        return ShardedMatrix(self.mesh, self.global_rows, self.global_cols,
                             [None if b is None else copy_block(padded_empty(tuple(b.shape), b.dtype, b.device), b)
                              for b in self.blocks], self.layout)


def _layout_grid(mesh: Mesh, layout: str) -> tuple[int, int]:
    if layout not in ("act", "weight"):
        raise ConfigError(f"unknown layout {layout!r}")
    return (mesh.r, mesh.c) if layout == "act" else (mesh.c, mesh.c)


def scatter(global_mat, mesh: Mesh, ws=None, category: str = "free", *, dtype: torch.dtype = F32,
            layout: str = "act", persistent: bool = False) -> ShardedMatrix:
    """Split a global matrix (numpy or torch) into device blocks (summa.py:59-77);
    ``persistent`` blocks come from ``mesh.persistent_empty`` (weight masters)."""
    g = torch.as_tensor(np.asarray(global_mat) if not isinstance(global_mat, torch.Tensor) else global_mat)
    if g.dim() != 2:
        raise ShapeError(f"scatter expects a 2-d matrix, got {g.dim()}-d")
    rows, cols = g.shape
    gr, gc = _layout_grid(mesh, layout)
    if rows % gr or cols % gc:
        raise ShapeError(f"matrix {rows}x{cols} not evenly divisible into {gr}x{gc} blocks")
    rb, cb = rows // gr, cols // gc
    s = ShardedMatrix(mesh, rows, cols, [None] * (gr * gc), layout)
    for k in range(gr * gc):
        i, j = divmod(k, gc)
        owner = s.owner(i, j)
        if not mesh.owns(owner):
            continue
        src = g[i * rb:(i + 1) * rb, j * cb:(j + 1) * cb]
        if persistent:
            blk = mesh.persistent_empty((rb, cb), dtype)
        else:
            blk = ws.empty(owner, (rb, cb), category, dtype=dtype) if ws is not None else \
                padded_empty((rb, cb), dtype, mesh.device(owner))
        blk.copy_(src.to(device=blk.device, dtype=dtype))
        s.blocks[k] = blk
    return s


def gather(s: ShardedMatrix) -> np.ndarray:
    """Reassemble the global matrix as float64 on the host (summa.py:80-88).

    Test-harness boundary; on the dist backend every process receives it.
    """
    gr, gc = s.grid
    rb, cb = s.block_rows, s.block_cols
    out = np.empty((s.global_rows, s.global_cols))
    mesh = s.mesh
    if mesh.is_local:
        for k, b in enumerate(s.blocks):
            i, j = divmod(k, gc)
            out[i * rb:(i + 1) * rb, j * cb:(j + 1) * cb] = b.detach().float().cpu().numpy()
        return out
    import torch.distributed as dist

    mine = {k: s.blocks[k].detach().float().cpu().numpy() for k in s.owned_indices()}
    parts = [None] * dist.get_world_size()
    dist.all_gather_object(parts, mine)
    for d in parts:
        for k, b in d.items():
            i, j = divmod(k, gc)
            out[i * rb:(i + 1) * rb, j * cb:(j + 1) * cb] = b
    return out


# ------------------------------------------------------------------ helpers

def as_bf16(mat: ShardedMatrix) -> ShardedMatrix:
    """The bf16 GEMM-operand view of a sharded matrix: itself, its attached
    ``bf16_twin`` (weights, fused-epilogue gradients) or a device cast."""
    if mat.dtype == BF16:
        return mat
    twin = getattr(mat, "bf16_twin", None)
    if twin is not None:
        return twin
    blocks = []
    for b in mat.blocks:
        if b is None:
            blocks.append(None)
            continue
        blocks.append(copy_block(padded_empty(tuple(b.shape), BF16, b.device), b))
    return ShardedMatrix(mat.mesh, mat.global_rows, mat.global_cols, blocks, mat.layout)


def _new_blocks(mesh: Mesh, ws, shape, category, dtype, layout="act"):
    gr, gc = _layout_grid(mesh, layout)
    out = [None] * (gr * gc)
    for k in range(gr * gc):
        i, j = divmod(k, gc)
        owner = mesh.flat(i, j) if layout == "act" else mesh.flat(i % mesh.r, j)
        if mesh.owns(owner):
            out[k] = ws.empty(owner, shape, category, dtype=dtype) if ws is not None else \
                padded_empty(shape, dtype, mesh.device(owner))
    return out


def _finish(mesh, acc_blocks, out_blocks, bias, c_blocks, act, aux_blocks, alpha=1.0):
    """Apply the GEMM epilogue to fp32 partial sums where it could not be fused."""
    for k, a in enumerate(acc_blocks):
        if a is None:
            continue
        K.epilogue(a, out_blocks[k], bias=None if bias is None else bias[k],
                   c=None if c_blocks is None else c_blocks[k], act=act,
                   aux=None if aux_blocks is None else aux_blocks[k], alpha=alpha)


def _reset_workspace(ws) -> None:
    """Every SUMMA product starts with an empty "workspace" arena (its staging and partial
    sums live for one product), as the reference resets it per step (summa.py:105, 129, 153)."""
    if ws is not None and hasattr(ws, "reset_all"):
        ws.reset_all("workspace")


def _check_pair(mesh, a, b, need_a, need_b, what):
    if a.grid != _layout_grid(mesh, need_a) or b.grid != _layout_grid(mesh, need_b):
        raise ConfigError(f"{what}: operands need layouts ({need_a}, {need_b}) on a {mesh.r}x{mesh.c} mesh")


# ------------------------------------------------------------------ SUMMA forms

def summa_ab(a: ShardedMatrix, b: ShardedMatrix, ws, out_category: str = "free", tag: str = "summa", *,
             out_dtype: torch.dtype = F32, bias=None, act: int = K.ACT_NONE, aux=None, resid=None,
             want_bf16: bool = False, colsum=None) -> ShardedMatrix:
    """C = A B in c steps: A(i,l) along row i, B(l,j) down column j, C_ij += A_il B_lj.

    summa.py:95-116. Optional fused epilogue (bias per output block, GELU with
    saved pre-activation ``aux``, residual ``resid`` added once) applied at the
    last step.
    """
    mesh = check_same_mesh(a, b)
    _reset_workspace(ws)
    if a.global_cols != b.global_rows:
        raise ShapeError(f"summa_ab inner dims differ: {a.global_cols} vs {b.global_rows}")
    _check_pair(mesh, a, b, "act", "weight", "summa_ab")
    steps = mesh.c
    m_b, k_b, n_b = a.block_rows, a.block_cols, b.block_cols
    a16, b16 = as_bf16(a), as_bf16(b)
    out = _new_blocks(mesh, ws, (m_b, n_b), out_category, out_dtype)
    out2 = _new_blocks(mesh, ws, (m_b, n_b), "free", BF16) if want_bf16 else None
    if resid is not None and (out_dtype != F32 or act != K.ACT_NONE):
        raise ConfigError("summa_ab: a residual is added to an fp32 linear output")
    # Accumulation across steps (and the residual) happens in place in fp32 via the
    # GEMM's TMA reduce-add stores. A fused epilogue that needs the complete sum
    # (GELU, bf16 output, column sums, bf16 copy) runs in the GEMM when there is a
    # single step, otherwise as one pass over the fp32 accumulator.
    fused_last = steps == 1 or (out_dtype == F32 and act == K.ACT_NONE and colsum is None and out2 is None)
    acc = out if fused_last else _new_blocks(mesh, ws, (m_b, n_b), "workspace", F32)
    # one step: the residual is the epilogue's C input (no copy); several steps: it
    # seeds the fp32 accumulator that the steps reduce-add into
    direct_resid = resid is not None and steps == 1
    for dev in mesh.local_devs:
        if resid is not None and not direct_resid:
            copy_block(acc[dev], resid.blocks[dev])
        elif steps > 1:
            K.zero(full_storage(acc[dev]))
    accumulate = (resid is not None and not direct_resid) or steps > 1
    # panels of step l+1 are in flight (double-buffered receive slots) while step l's
    # product runs; on the local backend the "broadcasts" alias the root's block
    a_rx, b_rx = _rx_slots(mesh, ws, (m_b, k_b)), _rx_slots(mesh, ws, (k_b, n_b))
    a_views, w_views = _peer_panels(mesh, a16, b16)

    def issue(l):
        return (mesh.bcast_row_async(l, a16.blocks, a_rx[l % 2], tag=tag, views=a_views),
                mesh.bcast_col_async(l % mesh.r, _weight_row(mesh, b16, l), b_rx[l % 2], tag=tag,
                                     views=None if w_views is None else w_views[l]))

    pend = issue(0)
    for l in range(steps):
        nxt = issue(l + 1) if l + 1 < steps else None
        a_pan, b_pan = pend[0].wait(), pend[1].wait()
        pend = nxt
        mesh.add_macs_all(m_b * k_b * n_b)
        last = l == steps - 1
        for dev in mesh.local_devs:
            c_in = acc[dev] if accumulate else (resid.blocks[dev] if direct_resid else None)
            if last and fused_last:
                K.gemm(a_pan[dev], b_pan[dev], out[dev], bias=None if bias is None else bias[dev], c=c_in, act=act,
                       aux=None if aux is None else aux.blocks[dev], out2=None if out2 is None else out2[dev],
                       colsum=None if colsum is None else colsum[dev])
            else:
                K.gemm(a_pan[dev], b_pan[dev], acc[dev], c=c_in)
    if not fused_last:
        for dev in mesh.local_devs:
            K.epilogue(acc[dev], out[dev], bias=None if bias is None else bias[dev], act=act,
                       aux=None if aux is None else aux.blocks[dev])
            if colsum is not None:
                K.colsum(out[dev], colsum[dev], accumulate=True)
            if out2 is not None:
                copy_block(out2[dev], out[dev])
    res = ShardedMatrix(mesh, a.global_rows, b.global_cols, out)
    if out2 is not None:
        res.bf16_twin = ShardedMatrix(mesh, a.global_rows, b.global_cols, out2)
    return res


def summa_abt(a: ShardedMatrix, b: ShardedMatrix, ws, out_category: str = "free", tag: str = "summa", *,
              out_dtype: torch.dtype = F32, act: int = K.ACT_NONE, aux=None, resid=None,
              colsum=None, ln_ctx=None) -> ShardedMatrix:
    """C = A B^T: B(l,j) down column j, A_ij B_lj^T, row-reduce to (i, l) (summa.py:119-140).

    ``ln_ctx`` (a LayerNormContext whose backward consumes C) lets a one-column
    local mesh accumulate that backward's row statistics in the GEMM epilogue;
    they are attached to the result as ``ln_stats`` (per-device [rows, 2]).
    """
    mesh = check_same_mesh(a, b)
    _reset_workspace(ws)
    if a.global_cols != b.global_cols:
        raise ShapeError(f"summa_abt contraction dims differ: {a.global_cols} vs {b.global_cols}")
    _check_pair(mesh, a, b, "act", "weight", "summa_abt")
    m_b, k_b, n_b = a.block_rows, a.block_cols, b.block_rows
    a16, b16 = as_bf16(a), as_bf16(b)
    out = _new_blocks(mesh, ws, (m_b, n_b), out_category, out_dtype)
    aux_b = None if aux is None else aux.blocks
    res_b = None if resid is None else resid.blocks
    fuse_ln = (ln_ctx is not None and mesh.is_local and mesh.c == 1 and out_dtype == F32 and act == K.ACT_NONE
               and resid is None and colsum is None)
    ln_stats = [None] * mesh.p
    if fuse_ln:
        for dev in mesh.local_devs:
            if ln_ctx.x.blocks[dev].dtype != F32:
                fuse_ln = False
    if mesh.is_local:
        # reduce fused into the accumulating GEMM chain, group-position order j = 0..c-1;
        # with c > 1 and GELU' the chain ends in fp32 and the epilogue runs as a pass
        # (the GEMM takes one global epilogue input at a time)
        split_epi = mesh.c > 1 and act != K.ACT_NONE
        for l in range(mesh.c):
            mesh.charge("broadcast", "col", l % mesh.r, n_b * k_b, tag)  # B(l, j) down column j
            mesh.charge("reduce", "row", l, m_b * n_b, tag)             # partials to (i, l)
            mesh.add_macs_all(m_b * k_b * n_b)
            for i in range(mesh.r):
                d = mesh.flat(i, l)
                chain = out[d] if mesh.c == 1 or (out_dtype == F32 and act == K.ACT_NONE) else \
                    ws_empty(ws, mesh, d, (m_b, n_b))
                if res_b is not None:
                    copy_block(chain, res_b[d])
                for j in range(mesh.c):
                    bt = b16.block(l, j).t()
                    prev = chain if (j > 0 or res_b is not None) else None
                    if j == mesh.c - 1 and fuse_ln:
                        ln_stats[d] = ws.empty(d, (m_b, 2), "free", dtype=F32, pad=False) if ws is not None \
                            else torch.empty((m_b, 2), dtype=F32, device=mesh.device(d))
                        K.zero(ln_stats[d])
                        K.gemm(a16.block(i, j), bt, out[d], ln_stats=(
                            ln_ctx.x.blocks[d], ln_ctx.gamma.for_position(mesh, d), ln_ctx.mean[d], ln_ctx.rstd[d],
                            ln_stats[d]))
                    elif j == mesh.c - 1 and not split_epi:
                        K.gemm(a16.block(i, j), bt, out[d], c=prev, act=act, aux=None if aux_b is None else aux_b[d],
                               colsum=None if colsum is None else colsum[d])
                    else:
                        K.gemm(a16.block(i, j), bt, chain, c=prev)
                if split_epi:
                    K.epilogue(chain, out[d], act=act, aux=None if aux_b is None else aux_b[d])
                    if colsum is not None:
                        K.colsum(out[d], colsum[d], accumulate=True)
        res = ShardedMatrix(mesh, a.global_rows, b.global_rows, out)
        if fuse_ln:
            res.ln_stats = ln_stats
        return res
    if mesh.peer is not None:
        return _abt_peer(mesh, ws, a16, b16, out, m_b, k_b, n_b, res_b, act, aux_b, colsum, tag, a.global_rows,
                         b.global_rows)
    # dist pipeline: B(l+1, j) arrives while step l's partial product runs, and step
    # l's row reduce overlaps step l+1's product (two partial-sum slots)
    acc = _new_blocks(mesh, ws, (m_b, n_b), "workspace", F32)
    b_rx = _rx_slots(mesh, ws, (n_b, k_b))
    part_slots = _rx_slots(mesh, ws, (m_b, n_b), F32)
    f = mesh.my_flat

    def issue(l):
        return mesh.bcast_col_async(l % mesh.r, _weight_row(mesh, b16, l), b_rx[l % 2], tag=tag)

    pend, red_prev = issue(0), None
    for l in range(mesh.c):
        nxt = issue(l + 1) if l + 1 < mesh.c else None
        b_pan = pend.wait()
        pend = nxt
        parts = [None] * mesh.p
        parts[f] = part_slots[l % 2]
        mesh.add_macs_all(m_b * k_b * n_b)
        K.gemm(a16.blocks[f], b_pan[f].t(), parts[f])
        red = mesh.reduce_row_async(l, parts, tag=tag)
        if red_prev is not None:
            red_prev.finish(acc)
        red_prev = red
    red_prev.finish(acc)
    _finish(mesh, acc, out, None, res_b, act, aux_b)
    if colsum is not None:
        for dev in mesh.local_devs:
            K.colsum(out[dev], colsum[dev], accumulate=True)
    return ShardedMatrix(mesh, a.global_rows, b.global_rows, out)


def summa_atb(a: ShardedMatrix, b: ShardedMatrix, ws, out_category: str = "free", tag: str = "summa", *,
              out_dtype: torch.dtype = F32, accumulate_into: ShardedMatrix | None = None,
              alpha: float = 1.0) -> ShardedMatrix:
    """C = A^T B: A(i,l) along row i, A_il^T B_ij, column-reduce to the owner of (l, j) (summa.py:143-164).

    ``accumulate_into`` adds the product to an existing weight-layout fp32
    matrix (gradient accumulation) instead of allocating the output; with
    ``alpha = -lr`` into the weight itself, that is the SGD step fused into the
    weight-gradient product (in-place TMA reduce-add, local meshes).
    """
    mesh = check_same_mesh(a, b)
    _reset_workspace(ws)
    if a.global_rows != b.global_rows:
        raise ShapeError(f"summa_atb contraction dims differ: {a.global_rows} vs {b.global_rows}")
    _check_pair(mesh, a, b, "act", "act", "summa_atb")
    m_b, t_b, n_b = a.block_cols, a.block_rows, b.block_cols
    a16, b16 = as_bf16(a), as_bf16(b)
    if accumulate_into is not None:
        out_mat = accumulate_into
        out = out_mat.blocks
    else:
        out = _new_blocks(mesh, ws, (m_b, n_b), out_category, out_dtype, layout="weight")
        out_mat = ShardedMatrix(mesh, a.global_cols, b.global_cols, out, "weight")
    acc_in = accumulate_into is not None
    if mesh.is_local:
        for l in range(mesh.c):
            mesh.charge("broadcast", "row", l, t_b * m_b, tag)      # A(i, l) along row i
            mesh.charge("reduce", "col", l % mesh.r, m_b * n_b, tag)  # partials to (l mod r, j)
            mesh.add_macs_all(m_b * t_b * n_b)
            for j in range(mesh.c):
                k = l * mesh.c + j
                chain = out[k] if out[k].dtype == F32 else ws_empty(ws, mesh, mesh.flat(l % mesh.r, j), (m_b, n_b))
                for i in range(mesh.r):
                    prev = chain if (i > 0 or acc_in) else None
                    dst = out[k] if i == mesh.r - 1 else chain
                    K.gemm(a16.block(i, l).t(), b16.block(i, j), dst, c=prev, alpha=alpha)
        return out_mat
    if mesh.peer is not None:
        return _atb_peer(mesh, ws, a16, b16, out_mat, m_b, t_b, n_b, acc_in, alpha, tag)
    if alpha != 1.0:
        raise ConfigError("summa_atb: alpha needs a local mesh or peer memory")
    # dist pipeline: A(i, l+1) arrives while step l's partial product runs, and step
    # l's column reduce overlaps step l+1's product
    a_rx = _rx_slots(mesh, ws, (t_b, m_b))
    part_slots = _rx_slots(mesh, ws, (m_b, n_b), F32)
    f = mesh.my_flat

    def issue(l):
        return mesh.bcast_row_async(l, a16.blocks, a_rx[l % 2], tag=tag)

    def dest_of(l):
        dest = [None] * mesh.p
        for j in range(mesh.c):
            o = out_mat.owner(l, j)
            if mesh.owns(o):
                dest[o] = out[l * mesh.c + j]
        return dest

    pend, red_prev = issue(0), None
    for l in range(mesh.c):
        nxt = issue(l + 1) if l + 1 < mesh.c else None
        a_pan = pend.wait()
        pend = nxt
        parts = [None] * mesh.p
        parts[f] = part_slots[l % 2]
        mesh.add_macs_all(m_b * t_b * n_b)
        K.gemm(a_pan[f].t(), b16.blocks[f], parts[f])
        red = (mesh.reduce_col_async(l % mesh.r, parts, tag=tag), dest_of(l))
        if red_prev is not None:
            red_prev[0].finish(red_prev[1], accumulate=acc_in)
        red_prev = red
    red_prev[0].finish(red_prev[1], accumulate=acc_in)
    return out_mat


def _abt_peer(mesh, ws, a16, b16, out, m_b, k_b, n_b, res_b, act, aux_b, colsum, tag, rows,
              cols) -> ShardedMatrix:
    """Dist AB^T with the row reduce fused into the GEMMs (peer memory, peer.py).

    Step l: B(l, j) arrives down column j (R2, double-buffered, step l+1 in flight);
    position (i, j)'s partial A(i,j) B(l,j)^T leaves its GEMM epilogue as a TMA
    reduce-add straight into the fp32 accumulator of the destination (i, l)
    (summa.py:128-139 reduce_row, mesh.py:458-475). No partial-sum buffers, reduce
    collectives or fold passes; two row barriers: accumulators zeroed before the
    first remote add, all adds landed before the epilogue reads them. The epilogue
    (residual, GELU', column sums) then runs on the destination's complete sum.
    """
    f = mesh.my_flat
    i = f // mesh.c
    acc, peers = mesh.peer.scratch("abt_acc", (m_b, n_b))
    K.zero(full_storage(acc))
    _, w_views = _peer_panels(mesh, None, b16)
    mesh.peer.barrier("all")  # accumulators zeroed, weight panels published / current
    b_rx = _rx_slots(mesh, ws, (n_b, k_b))

    def issue(l):
        return mesh.bcast_col_async(l % mesh.r, _weight_row(mesh, b16, l), b_rx[l % 2], tag=tag, views=w_views[l])

    pend = issue(0)
    for l in range(mesh.c):
        nxt = issue(l + 1) if l + 1 < mesh.c else None
        b_pan = pend.wait()
        pend = nxt
        mesh.charge("reduce", "row", l, m_b * n_b, tag)  # the reference's reduce_row, for the ledger
        mesh.add_macs_all(m_b * k_b * n_b)
        dst = peers[mesh.flat(i, l)]
        K.gemm(a16.blocks[f], b_pan[f].t(), dst, c=dst)
    mesh.peer.barrier("row")
    accs = [None] * mesh.p
    accs[f] = acc
    _finish(mesh, accs, out, None, res_b, act, aux_b)
    if colsum is not None:
        K.colsum(out[f], colsum[f], accumulate=True)
    return ShardedMatrix(mesh, rows, cols, out)


def _atb_peer(mesh, ws, a16, b16, out_mat, m_b, t_b, n_b, acc_in, alpha, tag) -> ShardedMatrix:
    """Dist A^T B with the column reduce fused into the GEMMs (peer memory).

    Step l: A(i, l) arrives along row i (R1); position (i, j)'s partial
    alpha A(i,l)^T B(i,j) is reduce-added by its GEMM epilogue into the owner of weight
    block (l, j), position (l mod r, j) (summa.py:152-163 reduce_col). When the
    destination blocks are themselves symmetric (weight masters: ``accumulate_into``
    with alpha = -lr is the SGD step fused into the weight-gradient product) the adds
    land in them directly; otherwise in a zeroed symmetric accumulator that the owner
    copies (or adds) into its output blocks after the closing column barrier.
    """
    f = mesh.my_flat
    i, j = divmod(f, mesh.c)
    r, c = mesh.r, mesh.c
    out = out_mat.blocks
    heap = mesh.peer.heap
    mine = [l for l in range(c) if l % r == i]
    direct = acc_in and all(heap.is_sym(out[l * c + j]) for l in mine)
    if not direct:
        acc, peers = mesh.peer.scratch("atb_acc", (c // r, m_b, n_b))
        K.zero(acc)
    a_views, _ = _peer_panels(mesh, a16, None)
    mesh.peer.barrier("all")  # accumulators zeroed, A panels published
    a_rx = _rx_slots(mesh, ws, (t_b, m_b))

    def issue(l):
        return mesh.bcast_row_async(l, a16.blocks, a_rx[l % 2], tag=tag, views=a_views)

    pend = issue(0)
    for l in range(c):
        nxt = issue(l + 1) if l + 1 < c else None
        a_pan = pend.wait()
        pend = nxt
        mesh.charge("reduce", "col", l % r, m_b * n_b, tag)
        mesh.add_macs_all(m_b * t_b * n_b)
        owner = mesh.flat(l % r, j)
        if direct:
            # the owner's block (l, j) is its (l // r)-th block of this matrix: SPMD allocation
            # put it at the offset of this position's own (l // r)-th block
            mine_same = out[(i + (l // r) * r) * c + j]
            dst = heap.peer(mine_same, owner) if owner != f else out[l * c + j]
        else:
            dst = peers[owner][l // r]
        K.gemm(a_pan[f].t(), b16.blocks[f], dst, c=dst, alpha=alpha)
    mesh.peer.barrier("col")
    if not direct:
        for l in mine:
            if acc_in:
                K.fold(out[l * c + j], [acc[l // r]], accumulate=True)
            else:
                copy_block(out[l * c + j], acc[l // r])
    return out_mat


def _peer_panels(mesh: Mesh, a16: ShardedMatrix | None, w16: ShardedMatrix | None):
    """Peer memory: publish this position's panel sources and return the views the
    pulls read. ``a`` (act layout): this position's one block, read along its row.
    ``w`` (weight layout): this position owns blocks (i + k r, j), k = 0..c/r-1; the
    root of step l, (l mod r, j), holds block (l, j) as its (l // r)-th block, at the
    offset of this position's own (l // r)-th block (SPMD) -> w_views[l]. Symmetric
    blocks (weight twins) are read in place; others are copied into a symmetric slot.
    (None, None) without peer memory; an AB / A^T B caller barriers after this."""
    if mesh.is_local or mesh.peer is None:
        return None, None
    f = mesh.my_flat
    i, j = divmod(f, mesh.c)
    a_views = None if a16 is None else mesh.publish("pan_a", a16.blocks[f])
    w_views = None
    if w16 is not None:
        r = mesh.r
        mine = [mesh.publish(f"pan_w{k}", w16.block(i + k * r, j)) for k in range(mesh.c // r)]
        w_views = [mine[l // r] for l in range(mesh.c)]
    if a16 is not None and w16 is not None:
        mesh.peer.barrier("all")
    return a_views, w_views


def _rx_slots(mesh: Mesh, ws, shape, dtype=BF16) -> list:
    """Two receive blocks for the double-buffered panel pipeline (dist backend only)."""
    if mesh.is_local:
        return [None, None]
    return [ws_empty(ws, mesh, mesh.my_flat, shape, dtype) for _ in range(2)]


def _weight_row(mesh: Mesh, w: ShardedMatrix, l: int) -> list:
    """Per-position list holding weight block (l, j) at its owner (l mod r, j)."""
    src = [None] * mesh.p
    for j in range(mesh.c):
        o = w.owner(l, j)
        if mesh.owns(o):
            src[o] = w.block(l, j)
    return src


def ws_empty(ws, mesh, dev, shape, dtype=F32):
    return ws.empty(dev, shape, "workspace", dtype=dtype) if ws is not None else \
        padded_empty(shape, dtype, mesh.device(dev))


def summa_ab_backward(c_grad, a, b, ws, a_out_category="free", b_out_category="free", tag="summa"):
    """Gradients of C = A B: (C_grad B^T, A^T C_grad) (summa.py:167-173)."""
    return (summa_abt(c_grad, b, ws, out_category=a_out_category, tag=tag),
            summa_atb(a, c_grad, ws, out_category=b_out_category, tag=tag))


def summa_abt_backward(c_grad, a, b, ws, a_out_category="free", b_out_category="free", tag="summa"):
    """Gradients of C = A B^T: (C_grad B, C_grad^T A) (summa.py:176-182)."""
    return (summa_ab(c_grad, b, ws, out_category=a_out_category, tag=tag),
            summa_atb(c_grad, a, ws, out_category=b_out_category, tag=tag))


def summa_atb_backward(c_grad, a, b, ws, a_out_category="free", b_out_category="free", tag="summa"):
    """Gradients of C = A^T B: (B C_grad^T, A C_grad) (summa.py:185-191)."""
    return (summa_abt(b, c_grad, ws, out_category=a_out_category, tag=tag),
            summa_ab(a, c_grad, ws, out_category=b_out_category, tag=tag))
