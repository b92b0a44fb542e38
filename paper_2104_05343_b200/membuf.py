"""Per-position device workspaces and the activation-checkpointed layer driver.

Mirrors the reference's arena contract (summagrid membuf.py:43-127, 174-266):
allocations are grouped by category ("workspace", "forward", "backward",
"param_grad", "param_grad_tied", "conjunction", "free", "replicated") with
per-position usage / high-water accounting and optional planned capacities
(BufferOverflowError). Memory itself comes from the torch CUDA caching
allocator on the mesh device; 2-D blocks get a 16-byte aligned row pitch so
they can feed TMA / vectorised kernels directly.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import Sequence

import numpy as np
import torch

from . import kernels as K
from .errors import BufferOverflowError, CheckpointMissingError, ConfigError

CATEGORIES = ("workspace", "forward", "backward", "param_grad", "param_grad_tied", "conjunction", "free",
              "replicated")

ALIGN_ELEMS = 8  # row pitch multiple: 16 bytes of bf16, 32 bytes of fp32


def padded_empty(shape: Sequence[int], dtype: torch.dtype, device) -> torch.Tensor:
    """Uninitialised tensor whose last-dim pitch is a multiple of 8 elements."""
    shape = tuple(int(s) for s in shape)
    if len(shape) < 2:
        n = shape[0] if shape else 1
        return torch.empty(-(-max(n, 1) // ALIGN_ELEMS) * ALIGN_ELEMS, dtype=dtype, device=device)[:n].view(shape)
    cols = shape[-1]
    ld = -(-max(cols, 1) // ALIGN_ELEMS) * ALIGN_ELEMS
    full = torch.empty(*shape[:-1], ld, dtype=dtype, device=device)
    return full[..., :cols]


def full_storage(view: torch.Tensor) -> torch.Tensor:
    """The contiguous padded [rows, pitch] region behind a padded 2-D view."""
    if view.is_contiguous():
        return view
    if view.dim() != 2 or view.stride(1) != 1:
        raise ConfigError("expected a padded 2-D block")
    return torch.as_strided(view, (view.shape[0], view.stride(0)), (view.stride(0), 1))


class Arena:
    """Accounting for one category on one position (membuf.py:43-67)."""

    def __init__(self, name: str, capacity: int | None = None) -> None:
        self.name = name
        self.capacity = capacity
        self.used = 0
        self.high_water = 0

    def charge(self, n: int) -> None:
        self.used += n
        if self.capacity is not None and self.used > self.capacity:
            raise BufferOverflowError(f"arena {self.name!r}: {self.used} scalars exceed planned {self.capacity}")
        self.high_water = max(self.high_water, self.used)

    def release(self, n: int) -> None:
        self.used = max(0, self.used - n)

    def reset(self) -> None:
        self.used = 0


class Workspace:
    """Per-position arena bundle (membuf.py:74-127)."""

    def __init__(self, p: int, capacities: dict | None = None, merge_fwd_bwd: bool = False,
                 device=None) -> None:
        caps = dict.fromkeys(CATEGORIES, None)
        if capacities:
            unknown = set(capacities) - set(CATEGORIES)
            if unknown:
                raise ConfigError(f"unknown workspace categories {sorted(unknown)}")
            caps.update(capacities)
        self.p = p
        self.merge_fwd_bwd = merge_fwd_bwd
        self.device = device if device is not None else (
            torch.device("cuda", torch.cuda.current_device()) if torch.cuda.is_available() else torch.device("cpu"))
        self.arenas: dict[str, list[Arena]] = {}
        for cat in CATEGORIES:
            if merge_fwd_bwd and cat == "backward":
                continue
            cap = caps[cat]
            if merge_fwd_bwd and cat == "forward":
                fc, bc = caps["forward"], caps["backward"]
                cap = None if fc is None or bc is None else fc + bc
            self.arenas[cat] = [Arena(cat, cap) for _ in range(p)]
        if merge_fwd_bwd:
            self.arenas["backward"] = self.arenas["forward"]

    def empty(self, dev: int, shape: Sequence[int], category: str = "free",
              dtype: torch.dtype = torch.float32, pad: bool = True) -> torch.Tensor:
        """Uninitialised block charged to ``category`` of position ``dev``.

        ``pad`` gives 2-D blocks a 16-byte aligned row pitch (GEMM / TMA
        operands); small packed buffers (per-row stats) use ``pad=False``.
        """
        if category not in self.arenas:
            raise ConfigError(f"unknown workspace category {category!r}")
        self.arenas[category][dev].charge(int(np.prod(shape)) if len(shape) else 1)
        if not pad:
            return torch.empty(tuple(shape), dtype=dtype, device=self.device)
        return padded_empty(shape, dtype, self.device)

    def alloc(self, dev: int, shape: Sequence[int], category: str = "free",
              dtype: torch.dtype = torch.float32) -> torch.Tensor:
        """Zero-filled aligned block (the reference's arenas hand out zeros, membuf.py:60)."""
        t = self.empty(dev, shape, category, dtype)
        K.zero(full_storage(t)) if t.dim() == 2 else K.zero(t)
        return t

    def reset_all(self, category: str) -> None:
        for a in self.arenas[category]:
            a.reset()

    def release_forward(self, dev: int, nscalars: int) -> None:
        if self.merge_fwd_bwd:
            self.arenas["forward"][dev].release(nscalars)

    def peak(self, category: str) -> np.ndarray:
        return np.array([a.high_water for a in self.arenas[category]], dtype=np.int64)

    def peaks(self) -> dict[str, np.ndarray]:
        return {cat: self.peak(cat) for cat in CATEGORIES if not (self.merge_fwd_bwd and cat == "backward")}


@dataclass(frozen=True)
class BufferPlan:
    """Planned per-position scalars for one layer (membuf.py:130-139)."""

    workspace_scalars: int
    forward_scalars: int
    backward_scalars: int
    param_grad_scalars: int
    conjunction_scalars: int


def plan_buffers(cfg, mesh_cfg) -> BufferPlan:
    """Per-position buffer plan of one layer on an r x c mesh (membuf.py:142-171 for r == c)."""
    r = getattr(mesh_cfg, "rows", 0) or mesh_cfg.q
    c = getattr(mesh_cfg, "cols", 0) or mesh_cfg.q
    p = r * c
    b, s, h = cfg.b, cfg.s, cfg.h
    bs = b * s
    if b % r or h % c or (bs * h) % p or (h * h) % p:
        raise ConfigError("model dimensions not divisible by the mesh")
    bsh_p = bs * h // p
    products = ((bs * h, 3 * h * h, 3 * bs * h), (bs * h, h * h, bs * h), (bs * h, 4 * h * h, 4 * bs * h),
                (4 * bs * h, 4 * h * h, bs * h))
    return BufferPlan(workspace_scalars=max((x + w + y) // p for x, w, y in products),
                      forward_scalars=9 * bsh_p, backward_scalars=7 * bsh_p,
                      param_grad_scalars=12 * h * h // p + 13 * (h // c), conjunction_scalars=bsh_p)


class CheckpointStore:
    """One saved layer input per layer (membuf.py:174-205)."""

    def __init__(self, p: int) -> None:
        self.p = p
        self._saved: dict = {}
        self.used = np.zeros(p, dtype=np.int64)
        self.high_water = np.zeros(p, dtype=np.int64)

    def save(self, layer_idx: int, x):
        from .summa import ShardedMatrix

        blocks = [None if b is None else _clone_block(b) for b in x.blocks]
        cp = ShardedMatrix(x.mesh, x.global_rows, x.global_cols, blocks, x.layout)
        self._saved[layer_idx] = cp
        for dev, b in enumerate(blocks):
            if b is not None:
                self.used[dev] += b.numel()
        np.maximum(self.high_water, self.used, out=self.high_water)
        return cp

    def get(self, layer_idx: int):
        try:
            return self._saved[layer_idx]
        except KeyError:
            raise CheckpointMissingError(f"no checkpoint saved for layer {layer_idx}") from None

    def discard(self, layer_idx: int) -> None:
        saved = self._saved.pop(layer_idx, None)
        if saved is not None:
            for dev, b in enumerate(saved.blocks):
                if b is not None:
                    self.used[dev] -= b.numel()

    def count(self) -> int:
        return len(self._saved)


def copy_block(dst: torch.Tensor, src: torch.Tensor) -> torch.Tensor:
    """dst[...] = src[...] for two aligned blocks of the same shape (device kernel)."""
    if tuple(dst.shape) != tuple(src.shape):
        raise ConfigError(f"copy_block shapes differ: {tuple(dst.shape)} vs {tuple(src.shape)}")
    fd, fs = (full_storage(dst), full_storage(src)) if dst.dim() == 2 else (dst, src)
    if fd.shape != fs.shape:
        raise ConfigError("copy_block needs matching row pitches")
    if fd.dtype == fs.dtype:
        K.fold(fd, [fs])
    else:
        K.cast(fs, fd)
    return dst


def _clone_block(b: torch.Tensor) -> torch.Tensor:
    return copy_block(padded_empty(tuple(b.shape), b.dtype, b.device), b)


def clone_to_conjunction(x, ws: Workspace):
    """Copy an activation-gradient shard into the reset conjunction arena (membuf.py:208-216)."""
    from .summa import ShardedMatrix

    ws.reset_all("conjunction")
    blocks = []
    for dev, b in enumerate(x.blocks):
        if b is None:
            blocks.append(None)
            continue
        blocks.append(copy_block(ws.empty(dev, tuple(b.shape), "conjunction", dtype=b.dtype), b))
    out = ShardedMatrix(x.mesh, x.global_rows, x.global_cols, blocks, x.layout)
    # fused by-products of the producer stay valid: the bf16 operand copy and the column sums
    for attr in ("bf16_twin", "colsum_parts"):
        if getattr(x, attr, None) is not None:
            setattr(out, attr, getattr(x, attr))
    return out


def checkpointed_forward(layers: Sequence, x0, store: CheckpointStore, ws: Workspace):
    """Keep only each layer's input, run the layer (membuf.py:219-234)."""
    x = x0
    for li, layer in enumerate(layers):
        x = store.save(li, x)
        ws.reset_all("forward")
        ws.reset_all("free")
        x, _ = layer.forward(x, ws)
    return x


def checkpointed_backward(layers: Sequence, loss_grad, store: CheckpointStore, ws: Workspace,
                          eager_update: bool = False, lr: float = 0.0):
    """Recompute each layer from its checkpoint, then backward (membuf.py:237-266)."""
    dy = loss_grad
    grads: list = [None] * len(layers)
    for li in reversed(range(len(layers))):
        x_in = store.get(li)
        ws.reset_all("forward")
        ws.reset_all("free")
        fwd = getattr(layers[li], "recompute_forward", layers[li].forward)
        _, saved = fwd(x_in, ws)
        ws.reset_all("backward")
        if eager_update and getattr(layers[li], "fused_sgd", False):
            dx, g = layers[li].backward(dy, saved, ws, lr=lr)  # weights updated by their dW products
        else:
            dx, g = layers[li].backward(dy, saved, ws)
        dy = clone_to_conjunction(dx, ws)
        store.discard(li)
        if eager_update:
            layers[li].apply_sgd(g, lr)
            ws.reset_all("param_grad")
        else:
            grads[li] = g
    return dy, grads
