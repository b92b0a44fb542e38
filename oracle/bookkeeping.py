"""Integer bookkeeping of the 2D partition, restated (oracle; test-only).

Generalises the reference's square q x q mesh to r x c (rows split the batch,
columns split the hidden size). For r == c every function reduces exactly to
the reference behaviour it cites; the r != c extension is the one documented
in DESIGN.md ("weight blocks (l, j) live on device (l mod r, j)").
"""

from __future__ import annotations

import numpy as np


def mesh_groups(r: int, c: int) -> tuple[list[list[int]], list[list[int]]]:
    """Row and column groups of flat ranks, flat = row*c + col (mesh.py:265-266, 281-282)."""
    rows = [[i * c + j for j in range(c)] for i in range(r)]
    cols = [[i * c + j for i in range(r)] for j in range(c)]
    return rows, cols


def bunched_tile(r: int, c: int, node_size: int) -> tuple[int, int]:
    """Most-square (a, b), a*b == node_size, a | r, b | c (mesh.py:230-245 for r == c).

    Ties keep the first candidate found with the smallest a, as the reference's
    strict ``<`` comparison does.
    """
    chosen = None
    for a in range(1, node_size + 1):
        if node_size % a:
            continue
        b = node_size // a
        if r % a or c % b:
            continue
        if chosen is None or abs(a - b) < abs(chosen[0] - chosen[1]):
            chosen = (a, b)
    if chosen is None:
        raise ValueError(f"node_size={node_size} cannot tile a {r}x{c} mesh")
    return chosen


def node_map(r: int, c: int, node_size: int, bunched: bool) -> list[int]:
    """Node id per flat rank: natural flat // node_size, or bunched tiles (mesh.py:267-275)."""
    if not bunched:
        return [f // node_size for f in range(r * c)]
    a, b = bunched_tile(r, c, node_size)
    return [(i // a) * (c // b) + (j // b) for i in range(r) for j in range(c)]


def act_block(x: np.ndarray, r: int, c: int, i: int, j: int) -> np.ndarray:
    """Activation-layout block (i, j): rows split r ways, columns c ways (summa.py:59-77)."""
    rb, cb = x.shape[0] // r, x.shape[1] // c
    return x[i * rb:(i + 1) * rb, j * cb:(j + 1) * cb]


def weight_block_owner(l: int, j: int, r: int, c: int) -> int:
    """Flat rank owning weight block (l, j) of a c x c weight grid: device (l mod r, j).

    For r == c this is device (l, j), the reference's scatter placement.
    """
    return (l % r) * c + j


def interleave_qkv(w: np.ndarray, parts: int) -> np.ndarray:
    """[Q|K|V] columns -> per column-part [Q_j|K_j|V_j] (layers.py:87-102)."""
    h = w.shape[-1] // 3
    hp = h // parts
    idx = np.concatenate([np.arange(comp * h + j * hp, comp * h + (j + 1) * hp)
                          for j in range(parts) for comp in range(3)])
    return w[..., idx]


def deinterleave_qkv(w: np.ndarray, parts: int) -> np.ndarray:
    """Inverse permutation of interleave_qkv (layers.py:105-115)."""
    h = w.shape[-1] // 3
    hp = h // parts
    idx = np.concatenate([np.arange(comp * h + j * hp, comp * h + (j + 1) * hp)
                          for j in range(parts) for comp in range(3)])
    inv = np.empty_like(idx)
    inv[idx] = np.arange(idx.size)
    return w[..., inv]


def token_block(tokens: np.ndarray, row: int, r: int) -> np.ndarray:
    """Flattened ids of the batch rows owned by mesh row ``row`` (layers.py:144-148)."""
    bb = tokens.shape[0] // r
    return tokens[row * bb:(row + 1) * bb].reshape(-1)


def v_padded(v: int, c: int) -> int:
    """Vocabulary rounded up to a multiple of the column count (layers.py:81-84)."""
    return -(-v // c) * c
