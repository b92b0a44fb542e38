"""The r x c device mesh: topology, rank placement and row/column collectives.

Drop-in for the reference's simulated mesh (summagrid mesh.py:40-531) with the
square q x q grid generalised to r x c (r | c; 1x1, 1x2, 2x2, 2x4 on one box).

Two execution back ends share one operator code path:

* ``local`` — one controller process drives all p mesh positions on one GPU
  (the reference's single-controller model, mesh.py:249). Every position owns
  its own blocks; "broadcasts" hand the root's block to the members (aliasing,
  the data already sits in the same HBM), reduces and all-reduces are
  rank-ordered fp32 folds on the device (sg_fold), so results are
  bit-reproducible like the reference's lockstep mode.
* ``dist`` — SPMD, one process per GPU (torch.distributed, NCCL over NVLink /
  NVSwitch; gloo for CPU-side tests). Each process owns the one mesh position
  placed on its rank; row and column communicators are created once.

Operators only use the "SPMD primitives" below (``bcast_row``, ``bcast_col``,
``reduce_row_into``, ``reduce_col_into``, ``allreduce_row``,
``allreduce_col``), which take per-position lists indexed by flat rank
(``None`` for positions this process does not own).
"""

from __future__ import annotations

import enum
import math
from collections import Counter
from dataclasses import dataclass
from typing import Callable, Sequence

import torch

from . import kernels as K
from .errors import ConfigError, MeshMismatchError, ShapeError
from .ledger import CommLedger


class Placement(enum.Enum):
    """Mapping of mesh positions onto nodes / GPU slots (mesh.py:40-44)."""

    NATURAL = "natural"
    BUNCHED = "bunched"


@dataclass(frozen=True)
class CostParams:
    """Kept for signature compatibility with the reference (mesh.py:47-58).

    The B200 build measures time instead of charging a beta/alpha model, but
    validates the values the same way.
    """

    beta: float = 1.0
    alpha: float = 0.0

    def __post_init__(self) -> None:
        if self.beta <= 0.0:
            raise ConfigError(f"beta must be > 0, got {self.beta}")
        if self.alpha < 0.0:
            raise ConfigError(f"alpha must be >= 0, got {self.alpha}")


@dataclass(frozen=True)
class MeshConfig:
    """Mesh shape and placement.

    ``MeshConfig(q)`` is the reference's square q x q mesh (mesh.py:61-81);
    ``MeshConfig(rows=r, cols=c)`` the r x c generalisation (r | c).
    """

    q: int = 0
    node_size: int = 1
    placement: Placement = Placement.NATURAL
    rows: int = 0
    cols: int = 0

    def __post_init__(self) -> None:
        r, c = self.rows, self.cols
        if r == 0 and c == 0:
            r = c = self.q
        elif self.q and (self.q != r or self.q != c):
            raise ConfigError(f"q={self.q} conflicts with rows={r}, cols={c}")
        if r < 1 or c < 1:
            raise ConfigError(f"mesh side q must be >= 1, got {self.q if self.q else (r, c)}")
        if c % r:
            raise ConfigError(f"mesh rows r={r} must divide columns c={c}")
        if self.node_size < 1:
            raise ConfigError(f"node_size must be >= 1, got {self.node_size}")
        if (r * c) % self.node_size:
            raise ConfigError(f"device count p={r * c} not divisible by node_size={self.node_size}")
        object.__setattr__(self, "rows", r)
        object.__setattr__(self, "cols", c)
        object.__setattr__(self, "q", r if r == c else 0)

    @property
    def p(self) -> int:
        return self.rows * self.cols


@dataclass(frozen=True)
class DeviceRank:
    row: int
    col: int
    node: int


def bunched_tile(r: int, c: int, node_size: int) -> tuple[int, int]:
    """Most-square (a, b) tile, a*b == node_size, a | r, b | c (mesh.py:230-245)."""
    best = None
    for a in range(1, node_size + 1):
        if node_size % a:
            continue
        b = node_size // a
        if r % a or c % b:
            continue
        if best is None or abs(a - b) < abs(best[0] - best[1]):
            best = (a, b)
    if best is None:
        raise ConfigError(f"no (rows x cols) tiling of node_size={node_size} fits a {r}x{c} mesh")
    return best


_MODES = ("lockstep", "threaded")


class Mesh:
    """The r x c grid. Drive it from one controller context per process."""

    def __init__(self, cfg: MeshConfig, cost: CostParams | None = None, mode: str = "lockstep", *,
                 backend: str = "local", device: torch.device | str | int | None = None,
                 peer: bool | None = None) -> None:
        if mode not in _MODES:
            raise ConfigError(f"unknown mesh mode {mode!r}")
        if backend not in ("local", "dist"):
            raise ConfigError(f"unknown mesh backend {backend!r}")
        self.cfg = cfg
        self.cost = cost or CostParams()
        self.mode = mode
        self.backend = backend
        self.r, self.c = cfg.rows, cfg.cols
        self.p = cfg.p
        self.q = cfg.q if cfg.q else None
        self._row_groups = [[i * self.c + j for j in range(self.c)] for i in range(self.r)]
        self._col_groups = [[i * self.c + j for i in range(self.r)] for j in range(self.c)]
        if cfg.placement is Placement.BUNCHED:
            ta, tb = bunched_tile(self.r, self.c, cfg.node_size)
            self._node = [(i // ta) * (self.c // tb) + (j // tb) for i in range(self.r) for j in range(self.c)]
        else:
            self._node = [f // cfg.node_size for f in range(self.p)]
        # slot = GPU ordinal / world rank of each position: nodes own consecutive
        # slots, positions inside a node in flat order
        seen: Counter = Counter()
        self._slot = []
        for f in range(self.p):
            n = self._node[f]
            self._slot.append(n * cfg.node_size + seen[n])
            seen[n] += 1
        self.stats: Counter = Counter()
        self.calls: Counter = Counter()  # torch.distributed calls actually issued (dist backend)
        self.ledger = CommLedger(self.p)
        self.peer = None
        self._closed = False
        if backend == "local":
            if device is None:
                device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                    else torch.device("cpu")
            self._device = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
            self.local_devs = list(range(self.p))
            self._groups = None
        else:
            import torch.distributed as dist

            if not dist.is_initialized():
                raise ConfigError("dist mesh needs torch.distributed initialised (one process per position)")
            if dist.get_world_size() != self.p:
                raise ConfigError(f"world size {dist.get_world_size()} != mesh size {self.p}")
            me = dist.get_rank()
            self.my_flat = self._slot.index(me)
            if device is None:
                device = torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() \
                    else torch.device("cpu")
            self._device = torch.device(device) if not isinstance(device, int) else torch.device("cuda", device)
            self.local_devs = [self.my_flat]
            # every process creates every group, in the same order
            rows = [dist.new_group([self._slot[f] for f in g]) if len(g) > 1 else None for g in self._row_groups]
            cols = [dist.new_group([self._slot[f] for f in g]) if len(g) > 1 else None for g in self._col_groups]
            self._groups = (rows, cols)
            # peer memory (CUDA IPC arenas + device barriers): the AB^T / A^T B reduces
            # become remote reduce-adds of the GEMM epilogues (peer.py); default on CUDA
            if peer is None:
                peer = self._device.type == "cuda" and self.p > 1
            if peer:
                if self._device.type != "cuda":
                    raise ConfigError("peer memory needs a CUDA device")
                from .peer import PeerNet

                self.peer = PeerNet(self)
            if self._device.type == "cuda" and self.p > 1 and self.peer is None and dist.get_backend() == "nccl":
                # the persistent GEMMs leave SMs to the NCCL kernels that move step l+1's
                # panels during step l's product (NCCL_MAX_NCHANNELS is set to match by bench.py)
                import os

                K.set_sm_reserve(int(os.environ.get("SG_SM_RESERVE", "8")))

    # ------------------------------------------------------------- topology
    def flat(self, row: int, col: int) -> int:
        return row * self.c + col

    def rank(self, flat: int) -> DeviceRank:
        return DeviceRank(row=flat // self.c, col=flat % self.c, node=self._node[flat])

    def node_of(self, flat: int) -> int:
        return self._node[flat]

    def slot_of(self, flat: int) -> int:
        """GPU ordinal (local backend on a full box) / world rank (dist backend)."""
        return self._slot[flat]

    def row_group(self, row: int) -> list[int]:
        return self._row_groups[row]

    def col_group(self, col: int) -> list[int]:
        return self._col_groups[col]

    def all_group(self) -> list[int]:
        return list(range(self.p))

    def nodes_in_group(self, group: Sequence[int]) -> set[int]:
        return {self._node[d] for d in group}

    def device(self, flat: int | None = None) -> torch.device:
        return self._device

    def persistent_empty(self, shape, dtype) -> torch.Tensor:
        """A long-lived block (weight masters): in the symmetric peer arena when the mesh
        has peer memory (so remote GEMM epilogues can reduce-add into it), else a
        padded device block."""
        if self.peer is not None:
            return self.peer.heap.empty(shape, dtype)
        from .membuf import padded_empty

        return padded_empty(shape, dtype, self._device)

    @property
    def is_local(self) -> bool:
        return self.backend == "local"

    def owns(self, flat: int) -> bool:
        return self.is_local or flat == self.my_flat

    # ------------------------------------------------------------- execution
    def each(self, fn: Callable[[int], None], devices: Sequence[int] | None = None) -> None:
        """Run fn(dev) for every position this process owns (mesh.py:304-324)."""
        for dev in (self.local_devs if devices is None else [d for d in devices if self.owns(d)]):
            fn(dev)

    def sync(self) -> None:
        if self._device.type == "cuda":
            torch.cuda.synchronize(self._device)

    def close(self) -> None:
        self._closed = True

    def __enter__(self) -> "Mesh":
        return self

    def __exit__(self, *exc) -> None:
        self.close()

    def _count(self, kind: str, tag: str) -> None:
        self.stats[(kind, tag)] += 1

    # ---- ledger (accounting only, ledger.py): the reference's cost model per collective
    @staticmethod
    def _numel(blocks) -> int:
        for b in blocks:
            if b is not None:
                return int(b.numel())
        return 0

    def _charge_group(self, kind: str, group: Sequence[int], root_pos: int, n: int, tag: str) -> None:
        if kind == "allreduce":
            self.ledger.charge_ring(group, n, self.cost.beta, tag, self.node_of)
        else:
            self.ledger.charge_tree(group, root_pos, n, self.cost.beta, tag, kind, self.node_of)

    def charge(self, kind: str, axis: str, root_pos: int, n: int, tag: str) -> None:
        """Count one collective call and charge it on every group of ``axis`` (row / col / all)."""
        self._count(kind, tag)
        groups = self._row_groups if axis == "row" else self._col_groups if axis == "col" else [self.all_group()]
        for g in groups:
            self._charge_group(kind, g, root_pos, n, tag)

    def add_macs(self, dev: int, count: int) -> None:
        self.ledger.macs[dev] += count

    def add_macs_all(self, count: int) -> None:
        """The same local product on every position (SUMMA steps)."""
        self.ledger.macs += count

    def collective_count(self, kind: str | None = None, tag: str | None = None) -> int:
        return sum(v for (k, t), v in self.stats.items() if (kind is None or k == kind) and (tag is None or t == tag))

    # ------------------------------------------------------------- SPMD primitives
    def _dist_group(self, axis: str, index: int):
        rows, cols = self._groups
        return rows[index] if axis == "row" else cols[index]

    def _bcast(self, axis: str, root: int, src: Sequence, shape, dtype, tag: str, views=None) -> list:
        """Each owned position receives the block of the group member at ``root``."""
        self.charge("broadcast", axis, root, int(math.prod(shape)) if shape else self._numel(src), tag)
        out: list = [None] * self.p
        if self.is_local:
            for f in self.local_devs:
                i, j = divmod(f, self.c)
                s = self.flat(i, root) if axis == "row" else self.flat(root, j)
                out[f] = src[s]
            return out
        import torch.distributed as dist

        f = self.my_flat
        i, j = divmod(f, self.c)
        s = self.flat(i, root) if axis == "row" else self.flat(root, j)
        group = self._dist_group(axis, i if axis == "row" else j)
        if group is None:
            out[f] = src[f]
            return out
        from .membuf import padded_empty

        buf = src[f] if f == s else padded_empty(shape, dtype, self._device)
        if self.peer is not None and f != s:
            if views is None:
                raise ConfigError("peer broadcast needs the root's published view")
            self.peer.transport.pull(buf, views[s]).wait()
            self.calls["peer_pull"] += 1
            out[f] = buf
            return out
        if self.peer is None or f != s:
            dist.broadcast(K._flat_storage(buf), src=self._slot[s], group=group)
            self.calls["broadcast"] += 1
        out[f] = buf
        return out

    # ---- asynchronous forms (the SUMMA pipeline): the transfer is enqueued on the
    # communicator's own stream, ordered after everything already enqueued on the
    # current stream, and ``wait()`` makes the current stream wait for it; step
    # l+1's panels are issued before step l's product so the two overlap.
    def _bcast_async(self, axis: str, root: int, src: Sequence, recv, tag: str, views=None) -> "Pending":
        self.charge("broadcast", axis, root, self._numel(src), tag)
        out: list = [None] * self.p
        if self.is_local:
            for f in self.local_devs:
                i, j = divmod(f, self.c)
                out[f] = src[self.flat(i, root) if axis == "row" else self.flat(root, j)]
            return Pending(out, [])
        import torch.distributed as dist

        f = self.my_flat
        i, j = divmod(f, self.c)
        s = self.flat(i, root) if axis == "row" else self.flat(root, j)
        group = self._dist_group(axis, i if axis == "row" else j)
        if group is None or (f == s and self.peer is not None):
            out[f] = src[f]
            return Pending(out, [])
        if self.peer is not None:
            # pull the root's published / symmetric block with a copy-engine copy (peer.py)
            if views is None:
                raise ConfigError("peer broadcast needs the root's published view")
            pend = self.peer.transport.pull(recv, views[s])
            self.calls["peer_pull"] += 1
            out[f] = recv
            pend.blocks = out
            return pend
        buf = src[f] if f == s else recv
        work = dist.broadcast(K._flat_storage(buf), src=self._slot[s], group=group, async_op=True)
        self.calls["broadcast"] += 1
        out[f] = buf
        return Pending(out, [work])

    def bcast_row_async(self, root_col: int, src: Sequence, recv, tag: str = "misc", views=None) -> "Pending":
        """Asynchronous bcast_row into the preallocated receive block ``recv`` (R1);
        ``views`` (peer memory): every position's view of the root's block."""
        if not 0 <= root_col < self.c:
            raise ConfigError(f"broadcast root column {root_col} out of range for c={self.c}")
        return self._bcast_async("row", root_col, src, recv, tag, views)

    def bcast_col_async(self, root_row: int, src: Sequence, recv, tag: str = "misc", views=None) -> "Pending":
        """Asynchronous bcast_col into the preallocated receive block ``recv`` (R2)."""
        if not 0 <= root_row < self.r:
            raise ConfigError(f"broadcast root row {root_row} out of range for r={self.r}")
        return self._bcast_async("col", root_row, src, recv, tag, views)

    def step_boundary(self) -> None:
        """End of a (graph-replayable) step on a peer-memory mesh: one whole-mesh barrier, so
        every member's reads of this step's published slots are done, and the slot
        parities restart. A CUDA graph of the step then replays with the slot order the
        eager step used; without the barrier, a name published an odd number of times per
        step would reuse its last slot for the next replay's first publish while a slower
        member may still be pulling from it."""
        if self.peer is None:
            return
        self.peer.barrier("all")
        self.peer.transport.reset_slots()

    def publish(self, name: str, block) -> list | None:
        """Peer memory: make this position's ``block`` readable by the mesh (a copy into a
        symmetric slot unless it already is symmetric); returns the views by flat rank.
        The caller orders the publish before the readers with a barrier."""
        if self.peer is None or block is None:
            return None
        self.calls["peer_publish"] += 1
        return self.peer.transport.publish(name, block)

    def sym_views(self, block, index_owner: int) -> list | None:
        """Peer memory: views, in every position, of the symmetric block that ``index_owner``
        holds at the same arena offset as this position's ``block`` (SPMD allocation)."""
        if self.peer is None or block is None:
            return None
        views = [None] * self.p
        views[index_owner] = self.peer.heap.peer(block, index_owner)
        return views

    def _reduce_async(self, axis: str, dest: int, parts: Sequence, tag: str) -> "Pending":
        """Start the group reduce of ``parts`` to group position ``dest``; ``finish``
        folds the sum into the destination's output block."""
        self.charge("reduce", axis, dest, self._numel(parts), tag)
        groups = self._row_groups if axis == "row" else self._col_groups
        if self.is_local:
            return Pending(list(parts), [], fold=[(g[dest], [parts[f] for f in g]) for g in groups])
        import torch.distributed as dist

        f = self.my_flat
        i, j = divmod(f, self.c)
        g = groups[i] if axis == "row" else groups[j]
        d = g[dest]
        group = self._dist_group(axis, i if axis == "row" else j)
        works = []
        if group is not None:
            flat = K._flat_storage(parts[f])
            if _reduce_ok(group, flat):
                works.append(dist.reduce(flat, dst=self._slot[d], group=group, async_op=True))
                self.calls["reduce"] += 1
            else:  # gloo reduce is CPU-only; all_reduce covers CUDA tensors
                works.append(dist.all_reduce(flat, group=group, async_op=True))
                self.calls["allreduce"] += 1
        return Pending(list(parts), works, fold=[(d, [parts[f]])] if f == d else [])

    def reduce_row_async(self, dest_col: int, parts: Sequence, tag: str = "misc") -> "Pending":
        if not 0 <= dest_col < self.c:
            raise ConfigError(f"reduce destination column {dest_col} out of range for c={self.c}")
        return self._reduce_async("row", dest_col, parts, tag)

    def reduce_col_async(self, dest_row: int, parts: Sequence, tag: str = "misc") -> "Pending":
        if not 0 <= dest_row < self.r:
            raise ConfigError(f"reduce destination row {dest_row} out of range for r={self.r}")
        return self._reduce_async("col", dest_row, parts, tag)

    def bcast_row(self, root_col: int, src: Sequence, shape=None, dtype=None, tag: str = "misc", views=None) -> list:
        """Position (i, j) gets src[(i, root_col)] (R1 panels, mesh.py:440-449)."""
        if not 0 <= root_col < self.c:
            raise ConfigError(f"broadcast root column {root_col} out of range for c={self.c}")
        return self._bcast("row", root_col, src, shape, dtype, tag, views)

    def bcast_col(self, root_row: int, src: Sequence, shape=None, dtype=None, tag: str = "misc", views=None) -> list:
        """Position (i, j) gets src[(root_row, j)] (R2 panels, mesh.py:451-456)."""
        if not 0 <= root_row < self.r:
            raise ConfigError(f"broadcast root row {root_row} out of range for r={self.r}")
        return self._bcast("col", root_row, src, shape, dtype, tag, views)

    def _reduce_into(self, axis: str, dest: int, parts: Sequence, out: Sequence, accumulate: bool, tag: str) -> None:
        self.charge("reduce", axis, dest, self._numel(parts), tag)
        if self.is_local:
            groups = self._row_groups if axis == "row" else self._col_groups
            for g in groups:
                d = g[dest]
                K.fold(out[d], [parts[f] for f in g], accumulate=accumulate)  # group-position order
            return
        import torch.distributed as dist

        f = self.my_flat
        i, j = divmod(f, self.c)
        g = self._row_groups[i] if axis == "row" else self._col_groups[j]
        d = g[dest]
        group = self._dist_group(axis, i if axis == "row" else j)
        part = parts[f]
        if self.peer is not None and group is not None:
            # the destination folds the group's published parts in group order (peer.py)
            self.peer.transport.reduce_into(axis, d, part, out[d] if f == d else None, accumulate)
            self.calls["peer_reduce"] += 1
            return
        if group is not None:
            flat = K._flat_storage(part)
            if _reduce_ok(group, flat):
                dist.reduce(flat, dst=self._slot[d], group=group)
                self.calls["reduce"] += 1
            else:  # gloo reduce is CPU-only; all_reduce covers CUDA tensors
                dist.all_reduce(flat, group=group)
                self.calls["allreduce"] += 1
        if f == d:
            K.fold(out[d], [part], accumulate=accumulate)

    def reduce_row_into(self, dest_col: int, parts: Sequence, out: Sequence, accumulate: bool = False,
                        tag: str = "misc") -> None:
        """out[(i, dest_col)] (+)= sum_j parts[(i, j)] (R3, mesh.py:458-475)."""
        if not 0 <= dest_col < self.c:
            raise ConfigError(f"reduce destination column {dest_col} out of range for c={self.c}")
        self._reduce_into("row", dest_col, parts, out, accumulate, tag)

    def reduce_col_into(self, dest_row: int, parts: Sequence, out: Sequence, accumulate: bool = False,
                        tag: str = "misc") -> None:
        """out[(dest_row, j)] (+)= sum_i parts[(i, j)] (R4, mesh.py:477-482)."""
        if not 0 <= dest_row < self.r:
            raise ConfigError(f"reduce destination row {dest_row} out of range for r={self.r}")
        self._reduce_into("col", dest_row, parts, out, accumulate, tag)

    def _allreduce(self, axis: str, bufs: Sequence, op: str, tag: str) -> None:
        if op not in ("sum", "max"):
            raise ConfigError(f"unknown all_reduce op {op!r}")
        self.charge("allreduce", axis, 0, self._numel(bufs), tag)
        if self.is_local:
            groups = self._row_groups if axis == "row" else self._col_groups
            for g in groups:
                if len(g) == 1:
                    continue
                first = bufs[g[0]]
                K.fold(first, [bufs[f] for f in g], op_max=(op == "max"))
                for f in g[1:]:
                    K.fold(bufs[f], [first])
            return
        import torch.distributed as dist

        f = self.my_flat
        i, j = divmod(f, self.c)
        group = self._dist_group(axis, i if axis == "row" else j)
        if group is None:
            return
        if self.peer is not None:
            self.peer.transport.allreduce(axis, K._flat_storage(bufs[f]), op)
            self.calls["peer_allreduce"] += 1
            return
        dist.all_reduce(K._flat_storage(bufs[f]), op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM,
                        group=group)
        self.calls["allreduce"] += 1

    def allreduce_row(self, bufs: Sequence, op: str = "sum", tag: str = "misc") -> None:
        """In place: every position of row i holds the fold of the row (R5-R7, mesh.py:501-504)."""
        self._allreduce("row", bufs, op, tag)

    def allreduce_col(self, bufs: Sequence, op: str = "sum", tag: str = "misc") -> None:
        """In place along columns (R8, mesh.py:506-508)."""
        self._allreduce("col", bufs, op, tag)

    def allreduce_all(self, bufs: Sequence, op: str = "sum", tag: str = "misc") -> None:
        """In place over every position of the mesh (the 1D baseline's ring all-reduce,
        baseline.py:128-202, mesh.py:510-513); position order on the local backend."""
        if op not in ("sum", "max"):
            raise ConfigError(f"unknown all_reduce op {op!r}")
        self.charge("allreduce", "all", 0, self._numel(bufs), tag)
        if self.is_local:
            first = bufs[0]
            K.fold(first, list(bufs), op_max=(op == "max"))
            for f in range(1, self.p):
                K.fold(bufs[f], [first])
            return
        import torch.distributed as dist

        if self.p > 1 and self.peer is not None:
            self.peer.transport.allreduce("all", K._flat_storage(bufs[self.my_flat]), op)
            self.calls["peer_allreduce"] += 1
        elif self.p > 1:
            dist.all_reduce(K._flat_storage(bufs[self.my_flat]),
                            op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
            self.calls["allreduce"] += 1

    # ------------------------------------------------ reference single-controller API
    # (local backend only: the caller holds every position's block, as in the reference)
    def _need_local(self) -> None:
        if not self.is_local:
            raise ConfigError("per-group reference collectives need the local (single-controller) backend")

    def broadcast_row(self, row: int, root_col: int, block: torch.Tensor, tag: str = "misc", ws=None,
                      category: str = "workspace") -> list[torch.Tensor]:
        """Staged copies of ``block`` for every member of ``row``, column order (mesh.py:440-449)."""
        self._need_local()
        if not 0 <= root_col < self.c:
            raise ConfigError(f"broadcast root column {root_col} out of range for c={self.c}")
        self._count("broadcast", tag)
        self._charge_group("broadcast", self._row_groups[row], root_col, int(block.numel()), tag)
        return [_staged_copy(block, ws, f, category) for f in self._row_groups[row]]

    def broadcast_col(self, col: int, root_row: int, block: torch.Tensor, tag: str = "misc", ws=None,
                      category: str = "workspace") -> list[torch.Tensor]:
        self._need_local()
        if not 0 <= root_row < self.r:
            raise ConfigError(f"broadcast root row {root_row} out of range for r={self.r}")
        self._count("broadcast", tag)
        self._charge_group("broadcast", self._col_groups[col], root_row, int(block.numel()), tag)
        return [_staged_copy(block, ws, f, category) for f in self._col_groups[col]]

    def _fold_blocks(self, blocks: Sequence[torch.Tensor], op: str) -> torch.Tensor:
        shape = tuple(blocks[0].shape)
        for b in blocks[1:]:
            if tuple(b.shape) != shape:
                raise ShapeError(f"reduce blocks differ in shape: {shape} vs {tuple(b.shape)}")
        srcs = [b.float().contiguous() for b in blocks]
        acc = torch.empty_like(srcs[0])
        K.fold(acc, srcs, op_max=(op == "max"))
        return acc

    def reduce_row(self, row: int, dest_col: int, blocks: Sequence[torch.Tensor], tag: str = "misc") -> torch.Tensor:
        self._need_local()
        if not 0 <= dest_col < self.c:
            raise ConfigError(f"reduce destination column {dest_col} out of range for c={self.c}")
        self._count("reduce", tag)
        self._charge_group("reduce", self._row_groups[row], dest_col, int(blocks[0].numel()), tag)
        return self._fold_blocks(blocks, "sum")

    def reduce_col(self, col: int, dest_row: int, blocks: Sequence[torch.Tensor], tag: str = "misc") -> torch.Tensor:
        self._need_local()
        if not 0 <= dest_row < self.r:
            raise ConfigError(f"reduce destination row {dest_row} out of range for r={self.r}")
        self._count("reduce", tag)
        self._charge_group("reduce", self._col_groups[col], dest_row, int(blocks[0].numel()), tag)
        return self._fold_blocks(blocks, "sum")

    def _all_reduce_blocks(self, group, blocks, op, tag):
        self._need_local()
        if op not in ("sum", "max"):
            raise ConfigError(f"unknown all_reduce op {op!r}")
        self._count("allreduce", tag)
        self._charge_group("allreduce", group, 0, int(blocks[0].numel()), tag)
        acc = self._fold_blocks(blocks, op)
        return [acc.clone() for _ in blocks]

    def all_reduce_row(self, row: int, blocks, op: str = "sum", tag: str = "misc"):
        return self._all_reduce_blocks(self._row_groups[row], blocks, op, tag)

    def all_reduce_col(self, col: int, blocks, op: str = "sum", tag: str = "misc"):
        return self._all_reduce_blocks(self._col_groups[col], blocks, op, tag)

    def all_reduce_all(self, blocks, op: str = "sum", tag: str = "misc"):
        return self._all_reduce_blocks(self.all_group(), blocks, op, tag)

    def local_matmul(self, dev: int, a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None,
                     accumulate: bool = False) -> torch.Tensor:
        """a @ b on one position's device with the tcgen05 GEMM (mesh.py:349-361)."""
        if a.shape[-1] != b.shape[0]:
            raise ShapeError(f"local matmul inner dims differ: {tuple(a.shape)} x {tuple(b.shape)}")
        if out is None:
            out = torch.empty(a.shape[0], b.shape[1], device=a.device, dtype=torch.float32)
        self.ledger.macs[dev] += int(a.shape[0]) * int(a.shape[1]) * int(b.shape[1])
        K.gemm(a.to(torch.bfloat16), b.to(torch.bfloat16), out, c=out if accumulate else None)
        return out


def _reduce_ok(group, t: torch.Tensor) -> bool:
    """dist.reduce is usable: NCCL, or gloo on CPU tensors (gloo's reduce is CPU-only)."""
    import torch.distributed as dist

    return dist.get_backend(group) == "nccl" or not t.is_cuda


class Pending:
    """An issued (possibly asynchronous) collective: ``blocks`` is the per-position
    result list, valid on the current stream after ``wait()``; for reduces,
    ``finish(out)`` also folds the group sum into the destination block (in
    group-position order on the local backend, mesh.py:464-466)."""

    def __init__(self, blocks: list, works: list, fold: list | None = None) -> None:
        self.blocks = blocks
        self.works = works
        self.fold = fold or []

    def wait(self) -> list:
        for w in self.works:
            w.wait()
        self.works = []
        return self.blocks

    def finish(self, out: Sequence, accumulate: bool = False) -> None:
        self.wait()
        for d, srcs in self.fold:
            if out[d] is not None:
                K.fold(out[d], srcs, accumulate=accumulate)
        self.fold = []


def _staged_copy(block: torch.Tensor, ws, dev: int, category: str) -> torch.Tensor:
    if ws is None:
        return block.clone()
    dst = ws.alloc(dev, tuple(block.shape), category, dtype=block.dtype)
    dst.copy_(block)
    return dst


def create_mesh(cfg: MeshConfig, cost: CostParams | None = None, mode: str = "lockstep", *,
                backend: str = "local", device=None, peer: bool | None = None) -> Mesh:
    """Build a mesh; raises ConfigError on an invalid config (mesh.py:516-518)."""
    return Mesh(cfg, cost=cost, mode=mode, backend=backend, device=device, peer=peer)


def check_same_mesh(*objs) -> Mesh:
    mesh = objs[0].mesh
    for o in objs[1:]:
        if o.mesh is not mesh:
            raise MeshMismatchError("operands live on different meshes")
    return mesh


def init_dist(backend: str = "nccl", timeout_s: float | None = None, **kwargs) -> None:
    """torch.distributed set-up for a dist mesh with failure detection: NCCL errors are
    raised asynchronously on the host (TORCH_NCCL_ASYNC_ERROR_HANDLING=1) and every
    collective carries a timeout (SG_DIST_TIMEOUT_S, default 600 s), so a dead or hung
    peer surfaces as an exception instead of a hang. The peer-memory step has its own
    device-side barrier timeout (PeerNet.check, ~10 s of spinning per barrier)."""
    import datetime
    import os

    import torch.distributed as dist

    if dist.is_initialized():
        return
    if backend == "nccl":
        os.environ.setdefault("TORCH_NCCL_ASYNC_ERROR_HANDLING", "1")
    t = timeout_s if timeout_s is not None else float(os.environ.get("SG_DIST_TIMEOUT_S", "600"))
    dist.init_process_group(backend, timeout=datetime.timedelta(seconds=t), **kwargs)


def mesh_for_world(world: int) -> MeshConfig:
    """The north-star grid for a GPU count: 1 -> 1x1, 2 -> 1x2, 4 -> 2x2, 8 -> 2x4."""
    table = {1: (1, 1), 2: (1, 2), 4: (2, 2), 8: (2, 4)}
    if world not in table:
        r = int(math.isqrt(world))
        while world % r:
            r -= 1
        table[world] = (r, world // r)
    r, c = table[world]
    return MeshConfig(rows=r, cols=c)
