"""Peer memory of the SPMD ("dist") mesh: symmetric device arenas mapped into every
process of the mesh through CUDA IPC, and device-side group barriers over them
(libsg ``sg_sym_alloc`` / ``sg_ipc_open`` / ``sg_peer_barrier``, csrc/sg_peer.cu).

The reference reduces the AB^T / A^T B partial products with a row / column
reduce per SUMMA step (summa.py:128-139, 152-163; mesh.py:458-482). Here every
position's GEMM reduce-adds its partial tile (TMA ``cp.reduce.async.bulk``)
directly into the destination position's accumulator, which lives in one of these
arenas: over NVLink between GPUs, in the same HBM for processes sharing a GPU.

Allocation is SPMD: every process allocates the same sequence of blocks, so a block
has the same arena and offset everywhere and only arena creation is collective
(one all-gather of IPC handles). The product path never allocates inside a
captured step: arenas are created by the warm-up steps.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from .errors import ConfigError, SummaGridError

ALIGN = 256
_KIND = {"row": 0, "col": 1, "all": 2}
_TYPESTR = {torch.float32: "<f4", torch.int32: "<i4", torch.int64: "<i8", torch.bfloat16: "<i2"}
# ~10 s at the B200's clock: a peer that never arrives turns into an error flag
# (PeerNet.check) instead of a hung device
BARRIER_TIMEOUT_CYCLES = 20_000_000_000


class _DevArray:
    """``__cuda_array_interface__`` over a raw device pointer (no ownership)."""

    def __init__(self, ptr: int, shape, strides, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "strides": tuple(strides), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 2}


def wrap(ptr: int, shape, dtype: torch.dtype, pitch: int | None = None) -> torch.Tensor:
    """A torch view of device memory at ``ptr`` (rows ``pitch`` elements apart for 2-D)."""
    if dtype not in _TYPESTR:
        raise ConfigError(f"peer memory: unsupported dtype {dtype}")
    es = torch.empty((), dtype=dtype).element_size()
    shape = tuple(int(s) for s in shape)
    # the storage spans whole padded rows (so full_storage() views stay in bounds); the
    # returned tensor is the [..., :cols] view of it
    full = shape[:-1] + (pitch,) if pitch is not None else shape
    strides, acc = [0] * len(full), es
    for k in reversed(range(len(full))):
        strides[k] = acc
        acc *= full[k]
    t = torch.as_tensor(_DevArray(ptr, full, strides, _TYPESTR[dtype]), device="cuda")
    if dtype == torch.bfloat16:
        t = t.view(dtype)
    return t[..., :shape[-1]] if pitch is not None else t


def _padded_pitch(shape) -> int | None:
    if len(shape) < 2:
        return None
    return -(-max(int(shape[-1]), 1) // 8) * 8


class SymHeap:
    """Bump allocator over symmetric arenas (same offsets on every process)."""

    def __init__(self, mesh, chunk_bytes: int = 1 << 28):
        self.mesh = mesh
        self.chunk = chunk_bytes
        self.arenas: list[tuple[int, int, list]] = []  # (local ptr, bytes, peer ptr by flat)
        self.used = 0
        self._cap = 0

    def _new_arena(self, nbytes: int) -> None:
        import torch.distributed as dist

        L = _lib.lib()
        size = max(nbytes, self.chunk)
        hsz = L.sg_ipc_handle_size()
        handle = ctypes.create_string_buffer(hsz)
        ptr = ctypes.c_void_p()
        _lib.check(L.sg_sym_alloc(size, ctypes.byref(ptr), handle), "sg_sym_alloc")
        mine = (self.mesh.my_flat, handle.raw, size)
        allh = [None] * dist.get_world_size()
        dist.all_gather_object(allh, mine)
        peers = [None] * self.mesh.p
        for flat, h, sz in allh:
            if sz != size:
                raise SummaGridError("peer arenas differ in size across processes (non-SPMD allocation)")
            if flat == self.mesh.my_flat:
                peers[flat] = ptr.value
            else:
                pp = ctypes.c_void_p()
                _lib.check(L.sg_ipc_open(ctypes.create_string_buffer(h, hsz), ctypes.byref(pp)), "sg_ipc_open")
                peers[flat] = pp.value
        self.arenas.append((ptr.value, size, peers))
        self.used, self._cap = 0, size

    def alloc(self, nbytes: int) -> tuple[int, int]:
        nbytes = -(-nbytes // ALIGN) * ALIGN
        if not self.arenas or self.used + nbytes > self._cap:
            self._new_arena(nbytes)
        a, off = len(self.arenas) - 1, self.used
        self.used += nbytes
        return a, off

    def empty(self, shape, dtype: torch.dtype) -> torch.Tensor:
        """A zero-initialised symmetric block (2-D blocks with a 16-byte aligned row pitch)."""
        shape = tuple(int(s) for s in shape)
        pitch = _padded_pitch(shape)
        es = torch.empty((), dtype=dtype).element_size()
        rows = 1
        for s in shape[:-1]:
            rows *= s
        nbytes = rows * (pitch if pitch is not None else (shape[-1] if shape else 1)) * es
        a, off = self.alloc(max(nbytes, es))
        return wrap(self.arenas[a][0] + off, shape, dtype, pitch)

    def is_sym(self, t: torch.Tensor) -> bool:
        return self._locate(t) is not None

    def _locate(self, t: torch.Tensor):
        ptr = t.data_ptr()
        for a, (base, size, _) in enumerate(self.arenas):
            if base <= ptr < base + size:
                return a, ptr - base
        return None

    def peer(self, t: torch.Tensor, flat: int) -> torch.Tensor:
        """The copy of symmetric block ``t`` held by mesh position ``flat`` (same view)."""
        loc = self._locate(t)
        if loc is None:
            raise ConfigError("peer(): tensor is not in a symmetric arena")
        a, off = loc
        if flat == self.mesh.my_flat:
            return t
        shape = tuple(t.shape)
        pitch = t.stride(-2) if t.dim() >= 2 else None
        return wrap(self.arenas[a][2][flat] + off, shape, t.dtype, pitch)


class PeerNet:
    """Symmetric arenas + device barriers of one dist mesh (CUDA only)."""

    def __init__(self, mesh):
        self.mesh = mesh
        self.heap = SymHeap(mesh)
        p = mesh.p
        self.pads = self.heap.empty((3 * p,), torch.int32)  # [row | col | all] x p slots, zeroed
        self.epoch = torch.zeros(3, dtype=torch.int32, device="cuda")
        self.err = torch.zeros(1, dtype=torch.int32, device="cuda")
        self._args: dict = {}
        self._scratch: dict = {}
        self._views: dict = {}
        self.barriers = 0
        self.transport = Transport(self)

    def _group(self, axis: str) -> list[int]:
        m = self.mesh
        i, j = divmod(m.my_flat, m.c)
        if axis == "row":
            return m.row_group(i)
        if axis == "col":
            return m.col_group(j)
        return m.all_group()

    def barrier(self, axis: str) -> None:
        """Stream-ordered barrier of this position's row / column / whole-mesh group: every
        member's earlier work (its remote reduce-adds included) precedes what follows."""
        group = self._group(axis)
        if len(group) == 1:
            return
        kind = _KIND[axis]
        if axis not in self._args:
            pads = self.heap.arenas[self._pad_arena()][2]
            off = self._pad_off() + kind * self.mesh.p * 4
            vals = [pads[f] + off for f in group] + list(group)
            self._args[axis] = torch.tensor(vals, dtype=torch.int64, device="cuda")
        L = _lib.lib()
        _lib.check(L.sg_peer_barrier(self._args[axis].data_ptr(), len(group), group.index(self.mesh.my_flat),
                                     self.epoch[kind:].data_ptr(), self.err.data_ptr(), BARRIER_TIMEOUT_CYCLES,
                                     torch.cuda.current_stream().cuda_stream), "sg_peer_barrier")
        self.barriers += 1

    def _pad_arena(self) -> int:
        return self.heap._locate(self.pads)[0]

    def _pad_off(self) -> int:
        return self.heap._locate(self.pads)[1]

    def scratch(self, name: str, shape, dtype: torch.dtype = torch.float32):
        """(local view, peer views by flat rank) of the symmetric region ``name`` shaped
        ``shape`` (2-D / 3-D with a padded row pitch). One region per name, grown on
        demand (SPMD: every process asks for the same sizes in the same order); ops on a
        stream reuse it one after another, separated by barriers."""
        shape = tuple(int(x) for x in shape)
        pitch = _padded_pitch(shape)
        es = torch.empty((), dtype=dtype).element_size()
        rows = 1
        for x in shape[:-1]:
            rows *= x
        need = rows * (pitch if pitch is not None else shape[-1]) * es
        base = self._scratch.get(name)
        if base is None or base[1] < need:
            a, off = self.heap.alloc(need)
            base = (a, need, off)
            self._scratch[name] = base
            self._views = {k: v for k, v in self._views.items() if k[0] != name}
        key = (name, shape, dtype)
        if key not in self._views:
            a, _, off = base
            arena = self.heap.arenas[a]
            self._views[key] = (wrap(arena[0] + off, shape, dtype, pitch),
                                [wrap(arena[2][f] + off, shape, dtype, pitch) for f in range(self.mesh.p)])
        return self._views[key]

    def check(self) -> None:
        """Raise if a barrier timed out (one host synchronisation)."""
        if int(self.err.item()):
            raise SummaGridError("peer barrier timed out: a mesh position did not arrive")


# ---------------------------------------------------------------- transfers over peer memory
class PeerPending:
    """A pull issued on the mesh's copy stream; ``wait()`` makes the current stream wait."""

    def __init__(self, blocks: list, event):
        self.blocks = blocks
        self.event = event

    def wait(self) -> list:
        if self.event is not None:
            torch.cuda.current_stream().wait_event(self.event)
            self.event = None
        return self.blocks


def _full(t: torch.Tensor) -> tuple[int, int]:
    """(pointer, bytes) of a block's whole padded storage (rows x pitch)."""
    if t.dim() >= 2:
        rows = 1
        for s in t.shape[:-1]:
            rows *= s
        return t.data_ptr(), rows * t.stride(-2) * t.element_size()
    return t.data_ptr(), t.numel() * t.element_size()


class Transport:
    """Panel broadcasts and small all-reduces of a dist mesh over its peer memory.

    * Broadcast (R1 / R2 panels, mesh.py:440-456): the root's block must be readable by
      the group: persistent symmetric blocks (weight masters / twins) are read where they
      are, other blocks are first published into a double-buffered symmetric slot
      (one local copy). Members then pull the panel with a copy-engine copy on the
      mesh's copy stream, ordered after everything already on the compute stream, so
      step l+1's panel moves while step l's product runs; the compute stream waits only
      for the panel it consumes.
    * All-reduce (R5-R8, mesh.py:484-513): each member publishes its buffer, one group
      barrier, then every member folds the group's buffers in group order
      (sg_peer_fold): the reference's rank-ordered fold, bit-identical on every member.
    A published slot is reused two publishes later on the same axis; the barrier of the
    publish in between orders every member's earlier reads before the overwrite.
    """

    def __init__(self, net: PeerNet):
        self.net = net
        self.stream = torch.cuda.Stream()
        self._parity: dict = {}
        self._ptrs: dict = {}

    def reset_slots(self) -> None:
        """Every name's next publish goes to slot 0 (after a whole-mesh barrier)."""
        self._parity.clear()

    def _slot(self, name: str, shape, dtype):
        k = self._parity.get(name, 0)
        self._parity[name] = k ^ 1
        return self.net.scratch(f"{name}.{k}", shape, dtype)

    def publish(self, name: str, block: torch.Tensor):
        """Copy a local block into its symmetric slot; returns peer views by flat rank."""
        if self.net.heap.is_sym(block):
            return [self.net.heap.peer(block, f) for f in range(self.net.mesh.p)]
        local, peers = self._slot(name, tuple(block.shape), block.dtype)
        dst, n = _full(local)
        src, n2 = _full(block)
        if n != n2:
            raise ConfigError("publish: blocks differ in pitch")
        _lib.check(_lib.lib().sg_copy_async(dst, src, n, torch.cuda.current_stream().cuda_stream), "sg_copy_async")
        return peers

    def pull(self, dst: torch.Tensor, src: torch.Tensor) -> PeerPending:
        """dst <- src (a peer's block) on the copy stream, after the compute stream's work so far."""
        cur = torch.cuda.current_stream()
        self.stream.wait_stream(cur)
        d, n = _full(dst)
        s, n2 = _full(src)
        if n != n2:
            raise ConfigError("pull: blocks differ in pitch")
        _lib.check(_lib.lib().sg_copy_async(d, s, n, self.stream.cuda_stream), "sg_copy_async")
        ev = torch.cuda.Event()
        ev.record(self.stream)
        return PeerPending([dst], ev)

    def _ptr_array(self, ptrs: list) -> torch.Tensor:
        """Device array of member pointers, cached by the pointers themselves (a slot region
        that grew has moved: its old arrays are never reused)."""
        key = tuple(ptrs)
        if key not in self._ptrs:
            self._ptrs[key] = torch.tensor(ptrs, dtype=torch.int64, device="cuda")
        return self._ptrs[key]

    def allreduce(self, axis: str, buf: torch.Tensor, op: str = "sum") -> None:
        """In place: buf = fold over this position's ``axis`` group, in group order."""
        group = self.net._group(axis)
        if len(group) == 1:
            return
        if buf.dtype != torch.float32 or not buf.is_contiguous():
            raise ConfigError("peer all-reduce: contiguous fp32 buffers")
        peers = self.publish(f"ar.{axis}", buf.view(-1))
        self.net.barrier(axis)
        srcs = self._ptr_array([peers[f].data_ptr() for f in group])
        _lib.check(_lib.lib().sg_peer_fold(buf.data_ptr(), srcs.data_ptr(), len(group), buf.numel(), 0,
                                           int(op == "max"), torch.cuda.current_stream().cuda_stream),
                   "sg_peer_fold")

    def reduce_into(self, axis: str, dest_flat: int, part: torch.Tensor, out, accumulate: bool) -> None:
        """out (+)= fold of the group's ``part`` blocks in group order, at ``dest_flat`` only."""
        group = self.net._group(axis)
        peers = self.publish(f"rd.{axis}", part)
        self.net.barrier(axis)
        if self.net.mesh.my_flat != dest_flat:
            return
        srcs = self._ptr_array([peers[f].data_ptr() for f in group])
        if out.stride(-2) != part.stride(-2):
            raise ConfigError("peer reduce: pitches differ")
        _, nbytes = _full(out)
        _lib.check(_lib.lib().sg_peer_fold(out.data_ptr(), srcs.data_ptr(), len(group), nbytes // 4,
                                           int(accumulate), 0, torch.cuda.current_stream().cuda_stream),
                   "sg_peer_fold")
