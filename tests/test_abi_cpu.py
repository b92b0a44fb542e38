"""The C-ABI library loads on a CPU-only host and exports every symbol of include/sg.h."""

import re
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def _declared() -> set[str]:
    text = (ROOT / "include" / "sg.h").read_text()
    return set(re.findall(r"^\s*(?:int|int64_t|const char\*)\s+(sg_\w+)\s*\(", text, flags=re.M))


def test_header_declares_the_path():
    names = _declared()
    for must in ("sg_gemm", "sg_ln_fwd", "sg_ln_bwd", "sg_xent_local", "sg_embed_fwd", "sg_sgd", "sg_fold"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2104_05343_b200 import _lib

    if not _lib._LIB_PATH.exists():
        pytest.skip("libsg.so not built (run __graft_entry__.build())")
    lib = _lib.lib()
    missing = [n for n in _declared() if not hasattr(lib, n)]
    assert not missing, missing
    assert set(_lib.SIGNATURES) == _declared(), "ctypes signatures out of sync with include/sg.h"
    assert b"sm_100a" in lib.sg_build_info()
    assert lib.sg_last_error() == b""


def test_no_cpu_fallback():
    """Kernels refuse host tensors instead of silently computing on the CPU."""
    import torch

    from paper_2104_05343_b200 import kernels
    from paper_2104_05343_b200.errors import ConfigError

    a = torch.zeros(8, 8, dtype=torch.bfloat16)
    with pytest.raises(ConfigError):
        kernels.gemm(a, a, torch.zeros(8, 8))
    with pytest.raises(ConfigError):
        kernels.bias_add(torch.zeros(8, 8), torch.zeros(8))
