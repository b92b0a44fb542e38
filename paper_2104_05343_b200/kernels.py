"""Per-device kernels: torch-tensor front end of the C ABI (include/sg.h).

Tensors are only used as device memory + streams; every computation below is a
call into libsg.so on the tensor's device and current CUDA stream.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import ACT_DGELU, ACT_GELU, ACT_NONE, DTYPE_BF16, DTYPE_F32, GemmArgs, check
from .errors import ConfigError, ShapeError

__all__ = ["gemm", "ACT_NONE", "ACT_GELU", "ACT_DGELU"]


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _require_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ConfigError("libsg operators take CUDA tensors (no CPU fallback)")


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return DTYPE_BF16
    if t.dtype == torch.float32:
        return DTYPE_F32
    raise ConfigError(f"unsupported dtype {t.dtype}")


def _batch(t: torch.Tensor, nbatch: int) -> tuple[int, int, int, int]:
    """(nb1, nb2, s1, s2) of the leading batch dims (0, 1 or 2 of them)."""
    if nbatch == 0:
        return 1, 1, 0, 0
    if nbatch == 1:
        return 1, t.shape[0], 0, t.stride(0)
    return t.shape[0], t.shape[1], t.stride(0), t.stride(1)


def gemm(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor, *, alpha: float = 1.0,
         bias: torch.Tensor | None = None, c: torch.Tensor | None = None, act: int = ACT_NONE,
         aux: torch.Tensor | None = None) -> torch.Tensor:
    """out = act(alpha * a @ b + bias + c) on the tcgen05 tensor cores.

    ``a`` [..., M, K] and ``b`` [..., K, N] are bf16 logical views; either may
    be a transposed view (unit stride on M / N instead of K), which selects the
    MN-major operand path instead of copying. ``out``/``c``/``aux`` are
    [..., M, N] with unit column stride. Up to two leading batch dims.
    """
    _require_cuda(a, b, out, bias, c, aux)
    if a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ConfigError("gemm operands must be bf16")
    nbd = a.dim() - 2
    if nbd < 0 or nbd > 2 or b.dim() != a.dim() or out.dim() != a.dim():
        raise ShapeError(f"gemm rank mismatch: {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(out.shape)}")
    M, K = a.shape[-2], a.shape[-1]
    K2, N = b.shape[-2], b.shape[-1]
    if K != K2 or tuple(out.shape[-2:]) != (M, N) or a.shape[:-2] != b.shape[:-2] or out.shape[:-2] != a.shape[:-2]:
        raise ShapeError(f"gemm shapes differ: {tuple(a.shape)} x {tuple(b.shape)} -> {tuple(out.shape)}")
    args = GemmArgs()
    args.M, args.N, args.K = M, N, K
    nb1, nb2, sa1, sa2 = _batch(a, nbd)
    args.nb1, args.nb2 = nb1, nb2
    # A operand: K-major (unit K stride) or MN-major (unit M stride)
    if a.stride(-1) == 1 and (a.stride(-2) >= K or M == 1):
        args.a_mn_major, args.lda = 0, max(a.stride(-2), K)
    elif a.stride(-2) == 1:
        args.a_mn_major, args.lda = 1, max(a.stride(-1), M)
    else:
        raise ShapeError("gemm: A needs unit stride along M or K")
    args.A, args.sa1, args.sa2 = a.data_ptr(), sa1, sa2
    _, _, sb1, sb2 = _batch(b, nbd)
    if b.stride(-2) == 1 and (b.stride(-1) >= K or N == 1):
        args.b_mn_major, args.ldb = 0, max(b.stride(-1), K)
    elif b.stride(-1) == 1:
        args.b_mn_major, args.ldb = 1, max(b.stride(-2), N)
    else:
        raise ShapeError("gemm: B needs unit stride along K or N")
    args.B, args.sb1, args.sb2 = b.data_ptr(), sb1, sb2
    if out.stride(-1) != 1:
        raise ShapeError("gemm: output needs unit column stride")
    _, _, sd1, sd2 = _batch(out, nbd)
    args.D, args.ldd, args.sd1, args.sd2, args.d_dtype = out.data_ptr(), out.stride(-2), sd1, sd2, _dtype_code(out)
    if c is not None:
        if tuple(c.shape) != tuple(out.shape) or c.stride(-1) != 1:
            raise ShapeError("gemm: C must match the output shape with unit column stride")
        _, _, sc1, sc2 = _batch(c, nbd)
        args.C, args.ldc, args.sc1, args.sc2, args.c_dtype = c.data_ptr(), c.stride(-2), sc1, sc2, _dtype_code(c)
    if bias is not None:
        if bias.dtype != torch.float32 or bias.numel() != N or not bias.is_contiguous():
            raise ShapeError("gemm: bias must be a contiguous fp32 vector of length N")
        args.bias = bias.data_ptr()
    if aux is not None:
        if tuple(aux.shape) != tuple(out.shape) or aux.dtype != torch.bfloat16 or aux.stride(-1) != 1:
            raise ShapeError("gemm: aux must be bf16 with the output shape")
        _, _, sx1, sx2 = _batch(aux, nbd)
        args.aux, args.ldx, args.sx1, args.sx2 = aux.data_ptr(), aux.stride(-2), sx1, sx2
    elif act == ACT_DGELU:
        raise ConfigError("gemm: DGELU epilogue needs the saved pre-activation (aux)")
    args.act = act
    args.alpha = alpha
    with torch.cuda.device(out.device):
        check(_lib.lib().sg_gemm(ctypes.byref(args), _stream(out)), "sg_gemm")
    return out
