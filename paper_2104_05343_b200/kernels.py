"""Per-device kernels: torch-tensor front end of the C ABI (include/sg.h).

Tensors are only used as device memory + streams; every computation below is a
call into libsg.so on the tensor's device and current CUDA stream.
"""

from __future__ import annotations

import ctypes

import torch

from . import _lib
from ._lib import (ACT_DGELU, ACT_GELU, ACT_NONE, DTYPE_BF16, DTYPE_F32, EPI_NORMAL, EPI_SOFTMAX,
                   EPI_SOFTMAX_BWD, GemmArgs, check)
from .errors import ConfigError, ShapeError

__all__ = ["gemm", "ACT_NONE", "ACT_GELU", "ACT_DGELU", "EPI_NORMAL", "EPI_SOFTMAX", "EPI_SOFTMAX_BWD"]


def _stream(t: torch.Tensor) -> int:
    # the current device's stream: peer-mapped tensors report their owner GPU as device
    return torch.cuda.current_stream().cuda_stream


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
         aux: torch.Tensor | None = None, out2: torch.Tensor | None = None, colsum: torch.Tensor | None = None,
         mode: int = EPI_NORMAL, rowvec: torch.Tensor | None = None, ln_stats=None) -> torch.Tensor:
    """out = act(alpha * a @ b + bias + c) on the tcgen05 tensor cores.

    ``a`` [..., M, K] and ``b`` [..., K, N] are bf16 logical views; either may
    be a transposed view (unit stride on M / N instead of K), which selects the
    MN-major operand path instead of copying. ``out``/``c``/``aux``/``out2``
    are [..., M, N] with unit column stride. Up to two leading batch dims.
    ``out2`` receives a bf16 copy of the result, ``colsum`` (fp32, [..., N]
    per batch, broadcast over size-1 batch strides) accumulates its column
    sums. ``mode`` selects the row-softmax epilogues (EPI_SOFTMAX: out =
    softmax(alpha * a @ b); EPI_SOFTMAX_BWD: out = aux * (acc - rowvec) *
    alpha with rowvec [..., M] = rowsum(acc * aux), e.g. rowsum(dO * O)).
    ``ln_stats = (x, gamma, mean, rstd, stats)`` accumulates the LayerNorm-
    backward row statistics of the fp32 output dy into ``stats`` [M, 2]
    (sum xhat * dy * gamma, sum dy * gamma); ``x`` is the LayerNorm input.
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
    if out2 is not None:
        if tuple(out2.shape) != tuple(out.shape) or out2.dtype != torch.bfloat16 or out2.stride(-1) != 1:
            raise ShapeError("gemm: out2 must be bf16 with the output shape")
        _, _, s21, s22 = _batch(out2, nbd)
        args.D2, args.ld2, args.s21, args.s22 = out2.data_ptr(), out2.stride(-2), s21, s22
    if colsum is not None:
        # colsum: [N] (summed over every batch) or [*batch, N] with size-1 dims broadcast
        if colsum.dtype != torch.float32 or colsum.stride(-1) != 1 or colsum.shape[-1] != N:
            raise ShapeError("gemm: colsum must be fp32 [..., N] with unit stride")
        lead = tuple(colsum.shape[:-1])
        if len(lead) not in (0, nbd):
            raise ShapeError("gemm: colsum batch dims must match the output's")
        cs = []
        for i, n_c in enumerate(lead):
            if n_c not in (1, out.shape[i]):
                raise ShapeError("gemm: colsum batch dim must be 1 or the output's")
            cs.append(colsum.stride(i) if n_c > 1 else 0)
        cs = [0] * (2 - len(cs)) + cs
        args.colsum, args.scs1, args.scs2 = colsum.data_ptr(), cs[0], cs[1]
    if rowvec is not None:
        if rowvec.dtype != torch.float32 or rowvec.shape[-1] != M or rowvec.stride(-1) != 1 or rowvec.dim() != nbd + 1:
            raise ShapeError("gemm: rowvec must be fp32 [*batch, M] with unit stride")
        _, _, sr1, sr2 = _batch(rowvec, nbd)
        args.rowvec, args.srv1, args.srv2 = rowvec.data_ptr(), sr1, sr2
    if ln_stats is not None:
        x, gamma, mean, rstd, stats = ln_stats
        if c is not None or bias is not None or act != ACT_NONE or nbd != 0 or out.dtype != torch.float32:
            raise ConfigError("gemm: LayerNorm statistics need an unbatched fp32 output without C / bias / act")
        if tuple(x.shape) != tuple(out.shape) or x.dtype != torch.float32 or x.stride(-1) != 1:
            raise ShapeError("gemm: the LayerNorm input must be fp32 with the output shape")
        if stats.dtype != torch.float32 or not stats.is_contiguous() or stats.numel() != 2 * M:
            raise ShapeError("gemm: LayerNorm statistics must be a contiguous fp32 [M, 2]")
        args.C, args.ldc, args.c_dtype = x.data_ptr(), x.stride(-2), DTYPE_F32
        args.ln_gamma, args.ln_mean, args.ln_rstd, args.ln_stats = (gamma.data_ptr(), mean.data_ptr(), rstd.data_ptr(),
                                                                    stats.data_ptr())
    args.mode = mode
    args.act = act
    args.alpha = alpha
    prof = _GEMM_PROFILE
    if prof is not None:
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
    # launched on the current device (``out`` may be a peer-mapped block of another GPU)
    check(_lib.lib().sg_gemm(ctypes.byref(args), _stream(out)), "sg_gemm")
    if prof is not None:
        e1.record(s)
        prof.append((2.0 * M * N * K * args.nb1 * args.nb2, e0, e1, (M, N, K, args.nb1 * args.nb2), _TAG[-1]))
    return out


_GEMM_PROFILE = None
_TAG = ["other"]


class tagged:
    """Label the GEMM launches inside the block (per-product roofline lists)."""

    def __init__(self, name: str):
        self.name = name

    def __enter__(self):
        _TAG.append(self.name)
        return self

    def __exit__(self, *exc):
        _TAG.pop()


class profile_gemms:
    """Record CUDA events around every sg_gemm launch on its stream.

    ``records`` holds (algorithmic flops, start event, end event, shape) per
    launch; ``summary()`` (after a synchronize) gives total flops, time and
    TFLOP/s of the GEMM kernel.
    """

    def __enter__(self):
        global _GEMM_PROFILE
        self.records = []
        _GEMM_PROFILE = self.records
        return self

    def __exit__(self, *exc):
        global _GEMM_PROFILE
        _GEMM_PROFILE = None

    def summary(self) -> dict:
        flops = sum(r[0] for r in self.records)
        ms = sum(r[1].elapsed_time(r[2]) for r in self.records)
        return {"launches": len(self.records), "flops": flops, "ms": ms,
                "tflops": flops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0}

    def by_tag(self) -> dict:
        """Per product label: launches, flops, ms and the distinct local shapes."""
        out: dict = {}
        for fl, e0, e1, shape, tag in self.records:
            d = out.setdefault(tag, {"launches": 0, "flops": 0.0, "ms": 0.0, "shapes": {}})
            d["launches"] += 1
            d["flops"] += fl
            d["ms"] += e0.elapsed_time(e1)
            d["shapes"][shape] = d["shapes"].get(shape, 0) + 1
        return out


def launch_count() -> int:
    """Kernels launched by libsg so far in this process."""
    return int(_lib.lib().sg_launch_count())


# ---------------------------------------------------------------- row kernels

def _p(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ConfigError("libsg operators take CUDA tensors (no CPU fallback)")
    return t.data_ptr()


def _dt(t):
    return DTYPE_F32 if t is None else _dtype_code(t)


def _rows2d(t: torch.Tensor) -> tuple[int, int, int]:
    """(rows, cols, ld) of a row-major 2-D view (leading dims flattened when contiguous)."""
    if t.dim() != 2:
        if not t.is_contiguous():
            raise ShapeError("row kernels need 2-D views or contiguous tensors")
        t = t.reshape(-1, t.shape[-1])
    if t.stride(-1) != 1 and t.shape[-1] > 1:
        raise ShapeError("row kernels need unit column stride")
    if t.shape[0] <= 1:  # the stride of a single row is irrelevant; report an aligned one
        return t.shape[0], t.shape[1], -(-t.shape[1] // 8) * 8
    return t.shape[0], t.shape[1], t.stride(0)


def _call(name: str, *args):
    check(getattr(_lib.lib(), name)(*args), name)


def ln_stats(x, stats):
    rows, cols, ldx = _rows2d(x)
    _call("sg_ln_stats", _p(x), _dt(x), rows, cols, ldx, _p(stats), _stream(x))


def ln_fwd(x, stats, h_total, eps, gamma, beta, y, mean, rstd):
    rows, cols, ldx = _rows2d(x)
    _, _, ldy = _rows2d(y)
    _call("sg_ln_fwd", _p(x), _dt(x), rows, cols, ldx, _p(stats), h_total, eps, _p(gamma), _p(beta), _p(y), _dt(y),
          ldy, _p(mean), _p(rstd), _stream(x))


def ln_bwd_stats(dy, x, mean, rstd, gamma, stats):
    rows, cols, lddy = _rows2d(dy)
    _, _, ldx = _rows2d(x)
    _call("sg_ln_bwd_stats", _p(dy), _dt(dy), lddy, _p(x), _dt(x), ldx, _p(mean), _p(rstd), _p(gamma), rows, cols,
          _p(stats), _stream(x))


def ln_bwd(dy, x, mean, rstd, gamma, stats, h_total, resid, dx, dx2=None, dgamma=None, dbeta=None, dsum=None):
    rows, cols, lddy = _rows2d(dy)
    _, _, ldx = _rows2d(x)
    ldr = _rows2d(resid)[2] if resid is not None else 0
    lddx = _rows2d(dx)[2]
    lddx2 = _rows2d(dx2)[2] if dx2 is not None else 0
    _call("sg_ln_bwd", _p(dy), _dt(dy), lddy, _p(x), _dt(x), ldx, _p(mean), _p(rstd), _p(gamma), rows, cols,
          _p(stats), h_total, _p(resid), _dt(resid), ldr, _p(dx), _dt(dx), lddx, _p(dx2), lddx2, _p(dgamma),
          _p(dbeta), _p(dsum), _stream(x))


def colsum(x, out, accumulate=False):
    rows, cols, ldx = _rows2d(x)
    _call("sg_colsum", _p(x), _dt(x), rows, cols, ldx, _p(out), int(accumulate), _stream(x))


def bias_add(x, bias):
    rows, cols, ldx = _rows2d(x)
    _call("sg_bias_add", _p(x), _dt(x), rows, cols, ldx, _p(bias), _stream(x))


def softmax_rows(s, p):
    rows, cols, lds = _rows2d(s)
    _, _, ldp = _rows2d(p)
    _call("sg_softmax_rows", _p(s), _dt(s), rows, cols, lds, _p(p), _dt(p), ldp, _stream(s))


def softmax_bwd(dp, p, scale, ds):
    rows, cols, lddp = _rows2d(dp)
    _, _, ldp = _rows2d(p)
    _, _, ldds = _rows2d(ds)
    _call("sg_softmax_bwd", _p(dp), _dt(dp), lddp, _p(p), _dt(p), ldp, rows, cols, scale, _p(ds), _dt(ds), ldds,
          _stream(dp))


def attn_rowdot(dO, O, n_heads, d, s, out):
    """out[b, h, t] = sum_j dO[b*s + t, h*d + j] * O[b*s + t, h*d + j]."""
    rows, _, ldo = _rows2d(dO)
    _, _, ldO = _rows2d(O)
    _call("sg_attn_rowdot", _p(dO), _dt(dO), ldo, _p(O), ldO, rows, n_heads, d, s, _p(out), _stream(dO))


def xent_local(logits, n_real, labels, col_lo, lmax, gmax, packed):
    rows, _, ldl = _rows2d(logits)
    _call("sg_xent_local", _p(logits), _dt(logits), rows, ldl, n_real, _p(labels), col_lo, _p(lmax), _p(gmax),
          _p(packed), _stream(logits))


def xent_rescale(lmax, gmax, packed):
    _call("sg_xent_rescale", lmax.numel(), _p(lmax), _p(gmax), _p(packed), _stream(lmax))


def xent_loss(gmax, packed, loss_rows, partial):
    _call("sg_xent_loss", gmax.numel(), _p(gmax), _p(packed), _p(loss_rows), _p(partial), _stream(gmax))


def xent_bwd(logits, n_real, labels, col_lo, gmax, packed, scale, dl):
    rows, ncols, ldl = _rows2d(logits)
    _, _, lddl = _rows2d(dl)
    _call("sg_xent_bwd", _p(logits), _dt(logits), rows, ldl, n_real, ncols, _p(labels), col_lo, _p(gmax),
          _p(packed), scale, _p(dl), _dt(dl), lddl, _stream(logits))


def embed_fwd(ids, lo, vb, table, out):
    _, hc, ldt = _rows2d(table)
    _, _, ldo = _rows2d(out)
    _call("sg_embed_fwd", _p(ids), ids.numel(), lo, vb, _p(table), _dt(table), ldt, hc, _p(out), _dt(out), ldo,
          _stream(out))


def embed_bwd(ids, lo, vb, dout, grad):
    _, hc, ldd = _rows2d(dout)
    _, _, ldg = _rows2d(grad)
    _call("sg_embed_bwd", _p(ids), ids.numel(), lo, vb, _p(dout), _dt(dout), ldd, hc, _p(grad), ldg, _stream(dout))


def sgd(w, w_bf16, g, lr):
    """w -= lr * g on fp32 master ``w`` (1-D or padded 2-D), refreshing the bf16 copy."""
    if w.dim() == 1:
        w2, g2, l2 = w.view(1, -1), g.view(1, -1), None if w_bf16 is None else w_bf16.view(1, -1)
    else:
        w2, g2, l2 = w, g, w_bf16
    rows, cols, ldw = _rows2d(w2)
    ldg = _rows2d(g2)[2]
    ldl = _rows2d(l2)[2] if l2 is not None else 0
    if tuple(g2.shape) != tuple(w2.shape) or (l2 is not None and tuple(l2.shape) != tuple(w2.shape)):
        raise ShapeError("sgd: parameter / gradient shapes differ")
    _call("sg_sgd", _p(w2), ldw, _p(l2), ldl, _p(g2), ldg, lr, rows, cols, _stream(w))


def sgd_multi(triples, lr):
    """w -= lr * g for every (w, w_bf16 | None, g) in one launch (multi-tensor SGD); g None:
    w was already updated (by its weight-gradient product), only its bf16 copy is refreshed."""
    items = []
    stream = None
    for w, wl, g in triples:
        if w.dim() == 1:
            w2, l2 = w.view(1, -1), None if wl is None else wl.view(1, -1)
            g2 = None if g is None else g.view(1, -1)
        else:
            w2, g2, l2 = w, g, wl
        if (g2 is not None and tuple(g2.shape) != tuple(w2.shape)) or \
                (l2 is not None and tuple(l2.shape) != tuple(w2.shape)):
            raise ShapeError("sgd: parameter / gradient shapes differ")
        if g2 is None and l2 is None:
            continue
        rows, cols, ldw = _rows2d(w2)
        it = _lib.SgdItem()
        it.w, it.w_bf16, it.g = _p(w2), _p(l2), _p(g2)
        it.ldw, it.ldl, it.ldg = ldw, (_rows2d(l2)[2] if l2 is not None else 0), \
            (_rows2d(g2)[2] if g2 is not None else 0)
        it.rows, it.cols = rows, cols
        items.append(it)
        stream = _stream(w) if stream is None else stream
    if not items:
        return
    arr = (_lib.SgdItem * len(items))(*items)
    _call("sg_sgd_multi", arr, len(items), lr, stream)


def cast(src, dst):
    if src.numel() != dst.numel() or not (src.is_contiguous() and dst.is_contiguous()):
        raise ShapeError("cast needs equal-size contiguous tensors")
    _call("sg_cast", _p(src), _dt(src), _p(dst), _dt(dst), src.numel(), _stream(dst))


def zero(t):
    if not t.is_contiguous():
        raise ShapeError("zero needs a contiguous tensor")
    _call("sg_zero", _p(t), t.numel() * t.element_size(), _stream(t))


def _flat_storage(t):
    """Contiguous 1-D view of a tensor, or of the padded rows behind a 2-D block view."""
    if t.is_contiguous():
        return t.reshape(-1)
    if t.dim() == 2 and t.stride(1) == 1 and t.stride(0) >= t.shape[1]:
        return torch.as_strided(t, (t.shape[0] * t.stride(0),), (1,))
    raise ShapeError("expected a contiguous tensor or a padded 2-D block")


def fold(dst, srcs, accumulate=False, op_max=False):
    """dst = [dst op] srcs[0] op srcs[1] ... in list order (op: + or max).

    Padded 2-D blocks with equal row pitch are folded over their full storage.
    """
    d = _flat_storage(dst)
    ss = []
    for s in srcs:
        f = _flat_storage(s)
        if f.numel() != d.numel() or s.dtype != dst.dtype or tuple(s.shape) != tuple(dst.shape):
            raise ShapeError("fold sources must match the destination")
        ss.append(f)
    # the kernel takes at most 8 sources per launch; longer groups (p > 8 meshes) fold
    # in list-order chunks, each chunk after the first accumulating into dst
    for k in range(0, max(1, len(ss)), _FOLD_MAX):
        chunk = ss[k:k + _FOLD_MAX]
        arr = (ctypes.c_void_p * max(1, len(chunk)))(*[s.data_ptr() for s in chunk])
        _call("sg_fold", _p(d), _dt(d), arr, len(chunk), d.numel(), int(accumulate or k > 0), int(op_max),
              _stream(d))


_FOLD_MAX = 8


def epilogue(x, out, *, bias=None, c=None, act=ACT_NONE, aux=None, alpha=1.0):
    """out = act(alpha*x + bias + c) for an fp32 x (the GEMM epilogue as a pass)."""
    rows, cols, ldx = _rows2d(x)
    ldc = _rows2d(c)[2] if c is not None else 0
    ldaux = _rows2d(aux)[2] if aux is not None else 0
    _, _, ldo = _rows2d(out)
    _call("sg_epilogue", _p(x), rows, cols, ldx, alpha, _p(bias), _p(c), _dt(c), ldc, act, _p(aux), ldaux, _p(out),
          _dt(out), ldo, _stream(x))


def dgelu(dact, mid, out, colsum=None):
    """out = dact * gelu'(mid) (out may alias dact); colsum += column sums of out."""
    rows, cols, lda = _rows2d(dact)
    _, _, ldm = _rows2d(mid)
    _, _, ldo = _rows2d(out)
    _call("sg_dgelu", _p(dact), lda, _p(mid), ldm, rows, cols, _p(out), _dt(out), ldo, _p(colsum), _stream(dact))


def qkv_grad_finish(dq_acc, dqkv, hb, colsum, q_only=False):
    """dqkv[:, :hb] = bf16(dq_acc); colsum += column sums of dqkv (fused; hb % 256 == 0),
    of its dQ columns only with ``q_only`` (dK / dV summed by the flash backward)."""
    rows, _, lddq = _rows2d(dq_acc)
    _, _, ldg = _rows2d(dqkv)
    _call("sg_qkv_grad_finish", _p(dq_acc), lddq, _p(dqkv), ldg, rows, hb, _p(colsum), hb if q_only else 3 * hb,
          _stream(dqkv))


def flash_attn_fwd(qkv, b, s, n_heads, d, out, lse=None):
    """Flash-style attention forward: qkv [b*s, 3*nh*d] block -> out [b*s, nh*d], lse [b, nh, s]."""
    _, _, ldq = _rows2d(qkv)
    _, _, ldo = _rows2d(out)
    _call("sg_flash_attn_fwd", _p(qkv), ldq, b, s, n_heads, d, _p(out), ldo, _p(lse), _stream(out))


def flash_attn_bwd(qkv, dout, lse, drow, b, s, n_heads, d, dq_acc, dqkv, kv_colsum=None):
    """dK, dV -> dqkv[:, nh*d:], dQ added into dq_acc (fp32, zeroed by the caller);
    ``kv_colsum`` ([2*nh*d] fp32) accumulates the column sums of dK, dV."""
    _, _, ldq = _rows2d(qkv)
    _, _, lddo = _rows2d(dout)
    _, _, lddq = _rows2d(dq_acc)
    _, _, ldg = _rows2d(dqkv)
    if kv_colsum is not None and (kv_colsum.dtype != torch.float32 or not kv_colsum.is_contiguous()
                                  or kv_colsum.numel() != 2 * n_heads * d):
        raise ShapeError("flash_attn_bwd: kv_colsum must be a contiguous fp32 [2 * nh * d]")
    _call("sg_flash_attn_bwd", _p(qkv), ldq, _p(dout), lddo, _p(lse), _p(drow), b, s, n_heads, d, _p(dq_acc), lddq,
          _p(dqkv), ldg, _p(kv_colsum), _stream(dqkv))


def check_ids(ids, v: int, flag):
    """flag (int32 [1]) |= 1 when any of ``ids`` lies outside [0, v) (sg_check_ids)."""
    _call("sg_check_ids", _p(ids), ids.numel(), v, _p(flag), _stream(flag))


def set_sm_reserve(n: int) -> None:
    """Leave ``n`` SMs free of the persistent GEMM grid (sg_set_sm_reserve)."""
    _call("sg_set_sm_reserve", int(n))


def gemm_sm_budget() -> int:
    return int(_lib.lib().sg_gemm_sm_budget())
