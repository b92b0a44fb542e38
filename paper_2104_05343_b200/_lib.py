"""ctypes binding of libsg.so (include/sg.h).

The library is mandatory: there is no CPU fallback for any operator. Loading
fails loudly when the in-tree build is missing; compute calls raise unless a
CUDA device is present.
"""

from __future__ import annotations

import ctypes
import os
from pathlib import Path

from .errors import ConfigError, ShapeError, SummaGridError

# SG_LIB_PATH: an alternative build of the same library (A/B timing of kernel variants)
_LIB_PATH = Path(os.environ.get("SG_LIB_PATH") or Path(__file__).resolve().parent / "libsg.so")

SG_OK, SG_ERR_SHAPE, SG_ERR_CONFIG, SG_ERR_CUDA = 0, 1, 2, 3
DTYPE_BF16, DTYPE_F32 = 0, 1
ACT_NONE, ACT_GELU, ACT_DGELU = 0, 1, 2
EPI_NORMAL, EPI_SOFTMAX, EPI_SOFTMAX_BWD = 0, 1, 2

i64 = ctypes.c_int64
i32 = ctypes.c_int32
vp = ctypes.c_void_p


class GemmArgs(ctypes.Structure):
    """Mirror of ``sg_gemm_args`` (include/sg.h)."""

    _fields_ = [
        ("M", i64), ("N", i64), ("K", i64),
        ("nb1", i64), ("nb2", i64),
        ("A", vp), ("lda", i64), ("sa1", i64), ("sa2", i64), ("a_mn_major", i32),
        ("B", vp), ("ldb", i64), ("sb1", i64), ("sb2", i64), ("b_mn_major", i32),
        ("D", vp), ("ldd", i64), ("sd1", i64), ("sd2", i64), ("d_dtype", i32),
        ("C", vp), ("ldc", i64), ("sc1", i64), ("sc2", i64), ("c_dtype", i32),
        ("bias", vp),
        ("aux", vp), ("ldx", i64), ("sx1", i64), ("sx2", i64),
        ("act", i32),
        ("alpha", ctypes.c_float),
        ("D2", vp), ("ld2", i64), ("s21", i64), ("s22", i64),
        ("colsum", vp), ("scs1", i64), ("scs2", i64),
        ("mode", i32),
        ("rowvec", vp), ("srv1", i64), ("srv2", i64),
        ("ln_gamma", vp), ("ln_mean", vp), ("ln_rstd", vp), ("ln_stats", vp),
    ]


class SgdItem(ctypes.Structure):
    """Mirror of ``sg_sgd_item`` (include/sg.h)."""

    _fields_ = [("w", vp), ("w_bf16", vp), ("g", vp), ("ldw", i64), ("ldl", i64), ("ldg", i64), ("rows", i64),
                ("cols", i64)]


# name -> (restype, argtypes); every symbol declared in include/sg.h
SIGNATURES: dict[str, tuple] = {
    "sg_gemm": (i32, [ctypes.POINTER(GemmArgs), vp]),
    "sg_ln_stats": (i32, [vp, i32, i64, i64, i64, vp, vp]),
    "sg_ln_fwd": (i32, [vp, i32, i64, i64, i64, vp, i64, ctypes.c_float, vp, vp, vp, i32, i64, vp, vp, vp]),
    "sg_ln_bwd_stats": (i32, [vp, i32, i64, vp, i32, i64, vp, vp, vp, i64, i64, vp, vp]),
    "sg_ln_bwd": (i32, [vp, i32, i64, vp, i32, i64, vp, vp, vp, i64, i64, vp, i64, vp, i32, i64, vp, i32, i64,
                        vp, i64, vp, vp, vp, vp]),
    "sg_colsum": (i32, [vp, i32, i64, i64, i64, vp, i32, vp]),
    "sg_bias_add": (i32, [vp, i32, i64, i64, i64, vp, vp]),
    "sg_softmax_rows": (i32, [vp, i32, i64, i64, i64, vp, i32, i64, vp]),
    "sg_softmax_bwd": (i32, [vp, i32, i64, vp, i32, i64, i64, i64, ctypes.c_float, vp, i32, i64, vp]),
    "sg_flash_attn_fwd": (i32, [vp, i64, i64, i64, i64, i64, vp, i64, vp, vp]),
    "sg_flash_attn_bwd": (i32, [vp, i64, vp, i64, vp, vp, i64, i64, i64, i64, vp, i64, vp, i64, vp, vp]),
    "sg_qkv_grad_finish": (i32, [vp, i64, vp, i64, i64, i64, vp, i64, vp]),
    "sg_attn_rowdot": (i32, [vp, i32, i64, vp, i64, i64, i64, i64, i64, vp, vp]),
    "sg_xent_local": (i32, [vp, i32, i64, i64, i64, vp, i64, vp, vp, vp, vp]),
    "sg_xent_rescale": (i32, [i64, vp, vp, vp, vp]),
    "sg_xent_loss": (i32, [i64, vp, vp, vp, vp, vp]),
    "sg_xent_bwd": (i32, [vp, i32, i64, i64, i64, i64, vp, i64, vp, vp, ctypes.c_float, vp, i32, i64, vp]),
    "sg_embed_fwd": (i32, [vp, i64, i64, i64, vp, i32, i64, i64, vp, i32, i64, vp]),
    "sg_embed_bwd": (i32, [vp, i64, i64, i64, vp, i32, i64, i64, vp, i64, vp]),
    "sg_check_ids": (i32, [vp, i64, i64, vp, vp]),
    "sg_sym_alloc": (i32, [i64, ctypes.POINTER(vp), vp]),
    "sg_sym_free": (i32, [vp]),
    "sg_ipc_open": (i32, [vp, ctypes.POINTER(vp)]),
    "sg_ipc_close": (i32, [vp]),
    "sg_ipc_handle_size": (i32, []),
    "sg_set_sm_reserve": (i32, [i32]),
    "sg_gemm_sm_budget": (i32, []),
    "sg_peer_barrier": (i32, [vp, i32, i32, vp, vp, i64, vp]),
    "sg_copy_async": (i32, [vp, vp, i64, vp]),
    "sg_peer_fold": (i32, [vp, vp, i32, i64, i32, i32, vp]),
    "sg_dgelu": (i32, [vp, i64, vp, i64, i64, i64, vp, i32, i64, vp, vp]),
    "sg_epilogue": (i32, [vp, i64, i64, i64, ctypes.c_float, vp, vp, i32, i64, i32, vp, i64, vp, i32, i64, vp]),
    "sg_sgd": (i32, [vp, i64, vp, i64, vp, i64, ctypes.c_float, i64, i64, vp]),
    "sg_sgd_multi": (i32, [ctypes.POINTER(SgdItem), i32, ctypes.c_float, vp]),
    "sg_cast": (i32, [vp, i32, vp, i32, i64, vp]),
    "sg_zero": (i32, [vp, i64, vp]),
    "sg_fold": (i32, [vp, i32, ctypes.POINTER(vp), i32, i64, i32, i32, vp]),
    "sg_device_sm_count": (i32, []),
    "sg_launch_count": (i64, []),
    "sg_build_info": (ctypes.c_char_p, []),
    "sg_last_error": (ctypes.c_char_p, []),
}

_lib = None


def lib():
    """Load libsg.so once; raise SummaGridError if the native build is absent."""
    global _lib
    if _lib is not None:
        return _lib
    if not _LIB_PATH.exists():
        raise SummaGridError(
            f"native library {_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`"
        )
    handle = ctypes.CDLL(str(_LIB_PATH), mode=os.RTLD_NOW | os.RTLD_GLOBAL)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(handle, name)
        fn.restype = res
        fn.argtypes = args
    _lib = handle
    return _lib


def check(rc: int, what: str) -> None:
    if rc == SG_OK:
        return
    msg = lib().sg_last_error().decode(errors="replace")
    text = f"{what}: {msg}" if msg else what
    if rc == SG_ERR_SHAPE:
        raise ShapeError(text)
    if rc == SG_ERR_CONFIG:
        raise ConfigError(text)
    raise SummaGridError(text)
