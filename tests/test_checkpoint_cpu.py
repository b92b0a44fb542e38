"""Model checkpoint file: the reference's binary format (model.py:64-79, 431-462),
checked byte-for-byte against a file written by the reference itself
(tests/golden/ckpt_small.bin, oracle/gen_golden.py)."""

from pathlib import Path

import numpy as np
import pytest

import paper_2104_05343_b200 as sg
from paper_2104_05343_b200.model import CKPT_MAGIC

GOLD = Path(__file__).parent / "golden" / "ckpt_small.bin"
CFG = dict(b=2, s=4, h=8, n=2, v=10, num_layers=1)


def test_writer_matches_reference_bytes(tmp_path):
    cfg = sg.ModelConfig(**CFG)
    params = sg.init_global_params(cfg, 3)
    out = tmp_path / "ckpt.bin"
    sg.save_checkpoint(out, cfg, params)
    assert out.read_bytes() == GOLD.read_bytes()


def test_reader_parses_reference_file():
    cfg, params, classifier = sg.load_checkpoint(GOLD)
    assert (cfg.b, cfg.s, cfg.h, cfg.n, cfg.v, cfg.num_layers) == tuple(CFG.values())
    assert cfg.eps == 1e-5 and classifier is False
    ref = sg.init_global_params(cfg, 3)
    assert list(params) == list(ref)
    for k in ref:
        np.testing.assert_array_equal(params[k], ref[k])


def test_round_trip_and_errors(tmp_path):
    cfg = sg.ModelConfig(**CFG)
    params = sg.init_global_params(cfg, 7)
    p = tmp_path / "a.bin"
    sg.save_checkpoint(p, cfg, params)
    cfg2, params2, _ = sg.load_checkpoint(p)
    assert cfg2 == cfg
    for k in params:
        np.testing.assert_array_equal(params2[k], params[k])
    bad = dict(params)
    bad["layers.0.w1"] = bad["layers.0.w1"][:, :3]
    with pytest.raises(sg.ShapeError):
        sg.save_checkpoint(tmp_path / "b.bin", cfg, bad)
    raw = bytearray(p.read_bytes())
    raw[0] ^= 0xFF
    (tmp_path / "c.bin").write_bytes(bytes(raw))
    with pytest.raises(sg.ConfigError, match="magic"):
        sg.load_checkpoint(tmp_path / "c.bin")
    (tmp_path / "d.bin").write_bytes(p.read_bytes()[:-8])
    with pytest.raises(sg.ConfigError, match="truncated"):
        sg.load_checkpoint(tmp_path / "d.bin")
    assert int.from_bytes(p.read_bytes()[:8], "little") == CKPT_MAGIC
