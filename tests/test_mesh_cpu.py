"""Host-side bookkeeping of the mesh and the model partition (no GPU needed).

Square meshes must match the reference bit-for-bit (golden fixtures made by the
real reference); the r x c generalisation is checked for its defining
properties.
"""

import json
from pathlib import Path

import numpy as np
import pytest

import paper_2104_05343_b200 as sg
from paper_2104_05343_b200 import layers

GOLD = Path(__file__).parent / "golden"


@pytest.fixture(scope="module")
def book():
    return json.loads((GOLD / "bookkeeping.json").read_text())


def _mesh(**kw):
    return sg.create_mesh(sg.MeshConfig(**kw), device="cpu")


def test_square_topology_matches_reference(book):
    for key, d in book["mesh"].items():
        q = int(key[1:])
        m = _mesh(q=q)
        assert [m.row_group(i) for i in range(q)] == d["rows"]
        assert [m.col_group(j) for j in range(q)] == d["cols"]
        for ns, nodes in d["natural_nodes"].items():
            mn = _mesh(q=q, node_size=int(ns))
            assert [mn.node_of(f) for f in range(q * q)] == nodes
        for ns, nodes in d["bunched_nodes"].items():
            if nodes is None:
                with pytest.raises(sg.ConfigError):
                    _mesh(q=q, node_size=int(ns), placement=sg.Placement.BUNCHED)
            else:
                mb = _mesh(q=q, node_size=int(ns), placement=sg.Placement.BUNCHED)
                assert [mb.node_of(f) for f in range(q * q)] == nodes


def test_rc_topology_and_slots():
    m = _mesh(rows=2, cols=4)
    assert m.p == 8 and m.q is None
    assert m.row_group(1) == [4, 5, 6, 7] and m.col_group(2) == [2, 6]
    assert m.rank(6) == sg.DeviceRank(row=1, col=2, node=6)
    for place in (sg.Placement.NATURAL, sg.Placement.BUNCHED):
        mm = _mesh(rows=2, cols=4, node_size=4, placement=place)
        slots = [mm.slot_of(f) for f in range(8)]
        assert sorted(slots) == list(range(8))
        for f in range(8):  # a node owns consecutive slots
            assert slots[f] // 4 == mm.node_of(f)
    mb = _mesh(rows=2, cols=4, node_size=4, placement=sg.Placement.BUNCHED)
    assert [mb.node_of(f) for f in range(8)] == [0, 0, 1, 1, 0, 0, 1, 1]  # 2x2 tiles
    assert sg.mesh_for_world(8) == sg.MeshConfig(rows=2, cols=4)
    assert sg.mesh_for_world(2) == sg.MeshConfig(rows=1, cols=2)


@pytest.mark.parametrize("kw", [dict(q=0), dict(q=2, node_size=0), dict(q=2, node_size=3), dict(rows=2, cols=3),
                                dict(q=2, rows=1, cols=2)])
def test_mesh_config_errors(kw):
    with pytest.raises(sg.ConfigError):
        sg.MeshConfig(**kw)


def test_mesh_mode_and_root_errors():
    with pytest.raises(sg.ConfigError):
        sg.create_mesh(sg.MeshConfig(q=2), mode="bogus", device="cpu")
    with pytest.raises(sg.ConfigError):
        sg.CostParams(beta=0)
    m = _mesh(q=2)
    with pytest.raises(sg.ConfigError):
        m.bcast_row(2, [None] * 4)
    with pytest.raises(sg.ConfigError):
        m.reduce_col_into(5, [None] * 4, [None] * 4)


def test_interleave_tokens_vpad_match_reference(book):
    for key, ref in book["interleave"].items():
        h, parts = map(int, key.split("_"))
        w = np.arange(3 * h, dtype=float)
        assert sg.interleave_qkv(w, parts).tolist() == ref
        assert np.array_equal(sg.deinterleave_qkv(sg.interleave_qkv(w, parts), parts), w)
    tok = np.arange(12).reshape(4, 3)
    for key, ref in book["token_block"].items():
        q = int(key[1:])
        assert [layers._token_block(tok, i, q).tolist() for i in range(q)] == ref
    cfg = sg.ModelConfig(b=4, s=2, h=8, n=2, v=37, num_layers=1)
    for key, ref in book["v_padded"].items():
        assert cfg.v_padded(int(key[1:])) == ref
    assert cfg.v_padded(sg.MeshConfig(rows=2, cols=4)) == 40


def test_model_config_validation():
    with pytest.raises(sg.ConfigError):
        sg.ModelConfig(b=2, s=2, h=10, n=3, v=4, num_layers=1)
    with pytest.raises(sg.ConfigError):
        sg.ModelConfig(b=0, s=2, h=8, n=2, v=4, num_layers=1)
    cfg = sg.ModelConfig(b=4, s=8, h=64, n=8, v=50, num_layers=2)
    cfg.validate_mesh(sg.MeshConfig(rows=2, cols=4))
    with pytest.raises(sg.ConfigError):
        cfg.validate_mesh(sg.MeshConfig(rows=2, cols=16))  # 16 heads needed
    with pytest.raises(sg.ConfigError):
        sg.ModelConfig(b=3, s=8, h=64, n=8, v=50, num_layers=1).validate_mesh(2)


def test_init_params_reference_stream():
    meta = json.loads((GOLD / "model.json").read_text())
    for name in ("small", "wide"):
        d = meta[name]
        cfg = sg.ModelConfig(*d["dims"])
        p = sg.init_global_params(cfg, d["seed"])
        for k, s in d["param_sums"].items():
            assert float(p[k].sum()) == s


def test_buffer_plan_matches_reference_formula():
    cfg = sg.ModelConfig(b=8, s=16, h=64, n=8, v=50, num_layers=2)
    plan = sg.plan_buffers(cfg, sg.MeshConfig(q=2))
    bsh_p = 8 * 16 * 64 // 4
    assert plan.forward_scalars == 9 * bsh_p and plan.backward_scalars == 7 * bsh_p
    assert plan.conjunction_scalars == bsh_p


def test_workspace_accounting():
    ws = sg.Workspace(4, capacities={"forward": 100}, device="cpu")
    ws.empty(1, (5, 10), "forward")
    assert ws.peak("forward").tolist() == [0, 50, 0, 0]
    with pytest.raises(sg.BufferOverflowError):
        ws.empty(1, (6, 10), "forward")
    ws.reset_all("forward")
    ws.empty(1, (10, 10), "forward")
    with pytest.raises(sg.ConfigError):
        sg.Workspace(1, capacities={"bogus": 1})
