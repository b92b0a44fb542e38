"""SUMMA AB / AB^T / A^T B and their backward forms on the mesh vs the oracle.

Inputs are bf16-representable so the check isolates the arithmetic (fp32
accumulate) from operand rounding; outputs are fp32.
"""

import numpy as np
import pytest

from tests._util import MESHES, bf16_round, mesh, rel

pytestmark = pytest.mark.gpu

TOL = 1e-4  # fp32 accumulate of exact bf16 operands


def _sg():
    import paper_2104_05343_b200 as sg

    return sg


@pytest.mark.parametrize("rc", MESHES + [(3, 3)])
def test_forms_match_oracle(rc):
    sg = _sg()
    r, c = rc
    m = mesh(r, c)
    rng = np.random.default_rng(100 + r * 10 + c)
    M, K, N = 48 * r, 32 * c, 40 * c
    a = bf16_round(rng.standard_normal((M, K)))
    b = bf16_round(rng.standard_normal((K, N)))
    bt = bf16_round(rng.standard_normal((N, K)))
    a2 = bf16_round(rng.standard_normal((M, N)))
    ws = sg.Workspace(m.p)
    A = sg.scatter(a, m)
    B = sg.scatter(b, m, layout="weight")
    BT = sg.scatter(bt, m, layout="weight")
    A2 = sg.scatter(a2, m)
    assert rel(sg.gather(sg.summa_ab(A, B, ws)), a @ b) < TOL
    assert rel(sg.gather(sg.summa_abt(A, BT, ws)), a @ bt.T) < TOL
    C = sg.summa_atb(A, A2, ws)
    assert C.layout == "weight" and C.grid == (c, c)
    assert rel(sg.gather(C), a.T @ a2) < TOL


@pytest.mark.parametrize("q", [1, 2, 3])
def test_golden_summa(q):
    """Reference-generated fixtures (oracle/gen_golden.py), q x q meshes."""
    from pathlib import Path

    sg = _sg()
    g = np.load(Path(__file__).parent / "golden" / "summa.npz")
    m = mesh(q, q)
    ws = sg.Workspace(m.p)
    a, b, bt, at, dc = (bf16_round(g[f"q{q}_{k}"]) for k in ("a", "b", "bt", "at", "dc"))
    A, B, BT, AT, DC = (sg.scatter(x, m) for x in (a, b, bt, at, dc))
    # the golden products were computed on the unrounded operands: bf16 operand
    # rounding is the dominant error here, hence the bf16 tolerance
    assert rel(sg.gather(sg.summa_ab(A, B, ws)), g[f"q{q}_ab"]) < 2e-2
    assert rel(sg.gather(sg.summa_abt(A, BT, ws)), g[f"q{q}_abt"]) < 2e-2
    assert rel(sg.gather(sg.summa_atb(AT, B, ws)), g[f"q{q}_atb"]) < 2e-2
    da, db = sg.summa_ab_backward(DC, A, B, ws)
    assert rel(sg.gather(da), g[f"q{q}_ab_da"]) < 2e-2
    assert rel(sg.gather(db), g[f"q{q}_ab_db"]) < 2e-2


@pytest.mark.parametrize("rc", [(1, 1), (2, 2), (2, 4)])
def test_backward_closure(rc):
    """Eqs. 1-3: every backward is expressed through the forward forms (summa.py:167-191)."""
    sg = _sg()
    r, c = rc
    m = mesh(r, c)
    rng = np.random.default_rng(7)
    M, K, N = 32 * r, 16 * c, 24 * c
    a = bf16_round(rng.standard_normal((M, K)))
    b = bf16_round(rng.standard_normal((K, N)))
    dc = bf16_round(rng.standard_normal((M, N)))
    ws = sg.Workspace(m.p)
    A, B, DC = sg.scatter(a, m), sg.scatter(b, m, layout="weight"), sg.scatter(dc, m)
    da, db = sg.summa_ab_backward(DC, A, B, ws)
    assert rel(sg.gather(da), dc @ b.T) < TOL
    assert rel(sg.gather(db), a.T @ dc) < TOL
    # C = A B^T with B in the weight layout: grads (dC B, dC^T A)
    bt = bf16_round(rng.standard_normal((N, K)))
    dct = bf16_round(rng.standard_normal((M, N)))
    BT, DCT = sg.scatter(bt, m, layout="weight"), sg.scatter(dct, m)
    ga, gb = sg.summa_abt_backward(DCT, A, BT, ws)
    assert rel(sg.gather(ga), dct @ bt) < TOL
    assert rel(sg.gather(gb), dct.T @ a) < TOL


def test_identity_and_errors():
    sg = _sg()
    m = mesh(2, 2)
    ws = sg.Workspace(m.p)
    rng = np.random.default_rng(3)
    a = bf16_round(rng.standard_normal((16, 16)))
    eye = np.eye(16)
    assert rel(sg.gather(sg.summa_ab(sg.scatter(a, m), sg.scatter(eye, m), ws)), a) < 1e-6
    with pytest.raises(sg.ShapeError):
        sg.summa_ab(sg.scatter(np.zeros((8, 4)), m), sg.scatter(np.zeros((8, 4)), m), ws)
    with pytest.raises(sg.ShapeError):
        sg.scatter(np.zeros((5, 4)), m)
    other = mesh(2, 2)
    with pytest.raises(sg.MeshMismatchError):
        sg.summa_ab(sg.scatter(a, m), sg.scatter(a, other), ws)


def test_collective_counts_per_form():
    """c steps of broadcasts, and reduces only in the AB^T / A^T B forms."""
    sg = _sg()
    m = mesh(2, 2)
    ws = sg.Workspace(m.p)
    a = np.ones((8, 8))
    A = sg.scatter(a, m)
    m.stats.clear()
    sg.summa_ab(A, A, ws)
    assert m.collective_count("broadcast") == 2 * m.c and m.collective_count("reduce") == 0
    m.stats.clear()
    sg.summa_abt(A, A, ws)
    assert m.collective_count("reduce") == m.c
