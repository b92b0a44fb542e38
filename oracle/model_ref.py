"""Serial float64 restatement of the reference transformer (oracle; test-only).

Math follows the reference exactly:
  * parameter draw order and ranges — model.py:97-119, dense.py:22-35
  * data stream (tokens then labels from PCG64(seed+1)) — cli.py:90-94
  * pre-norm layer y1 = x + Attn(LN1 x); out = y1 + MLP(LN2 y1) — layers.py:674-726
  * one-pass LayerNorm variance E[x^2] - E[x]^2, eps 1e-5 — layers.py:274-305
  * unmasked softmax(Q K^T / sqrt(d)) V per head — layers.py:393-416
  * tanh GELU and its exact derivative — dense.py:52-64
  * tied lm-head logits x table^T and mean-over-(b*s) cross entropy — layers.py:515-608
  * backward by explicit matrix calculus — oracle.py:158-205, layers.py:310-351, 424-508
The code is organised as a forward "tape" of per-layer records consumed in
reverse by ``serial_backward``.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

_C = math.sqrt(2.0 / math.pi)
_A = 0.044715


@dataclass(frozen=True)
class RefConfig:
    b: int
    s: int
    h: int
    n: int
    v: int
    num_layers: int
    eps: float = 1e-5

    @property
    def d(self) -> int:
        return self.h // self.n


def make_rng(seed: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(seed))


LAYER_KEYS = ("ln1_gamma", "ln1_beta", "w_qkv", "b_qkv", "w_dense", "b_dense",
              "ln2_gamma", "ln2_beta", "w1", "b1", "w2", "b2")


def init_params(cfg: RefConfig, seed: int) -> dict[str, np.ndarray]:
    """Uniform [-1/sqrt(h), 1/sqrt(h)) weights in draw order; identity vectors."""
    rng = make_rng(seed)
    lim = 1.0 / math.sqrt(cfg.h)
    h = cfg.h
    out = {"table": rng.uniform(-lim, lim, size=(cfg.v, h))}
    for i in range(cfg.num_layers):
        p = f"layers.{i}."
        out[p + "w_qkv"] = rng.uniform(-lim, lim, size=(h, 3 * h))
        out[p + "w_dense"] = rng.uniform(-lim, lim, size=(h, h))
        out[p + "w1"] = rng.uniform(-lim, lim, size=(h, 4 * h))
        out[p + "w2"] = rng.uniform(-lim, lim, size=(4 * h, h))
        for g in ("ln1_gamma", "ln2_gamma"):
            out[p + g] = np.ones(h)
        for z, width in (("ln1_beta", h), ("ln2_beta", h), ("b_qkv", 3 * h), ("b_dense", h),
                         ("b1", 4 * h), ("b2", h)):
            out[p + z] = np.zeros(width)
    return out


def sample_data(cfg: RefConfig, seed: int) -> tuple[np.ndarray, np.ndarray]:
    rng = make_rng(seed + 1)
    tokens = rng.integers(0, cfg.v, size=(cfg.b, cfg.s))
    labels = rng.integers(0, cfg.v, size=(cfg.b, cfg.s))
    return tokens, labels


# ----------------------------------------------------------------- pointwise

def gelu(x: np.ndarray) -> np.ndarray:
    return 0.5 * x * (1.0 + np.tanh(_C * (x + _A * x ** 3)))


def gelu_grad(x: np.ndarray) -> np.ndarray:
    t = np.tanh(_C * (x + _A * x ** 3))
    return 0.5 * (1.0 + t) + 0.5 * x * (1.0 - t * t) * _C * (1.0 + 3.0 * _A * x * x)


def softmax_last(x: np.ndarray) -> np.ndarray:
    e = np.exp(x - x.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


# ----------------------------------------------------------------- blocks

def layernorm(x, gamma, beta, eps):
    h = x.shape[-1]
    mean = x.sum(-1) / h
    var = (x * x).sum(-1) / h - mean * mean
    rstd = 1.0 / np.sqrt(var + eps)
    xhat = (x - mean[:, None]) * rstd[:, None]
    return xhat * gamma + beta, (xhat, rstd, mean, gamma)


def layernorm_grad(dy, rec):
    xhat, rstd, _, gamma = rec
    h = dy.shape[-1]
    g = dy * gamma
    m_xg = (xhat * g).sum(-1) / h
    m_g = g.sum(-1) / h
    dx = rstd[:, None] * (g - m_g[:, None] - xhat * m_xg[:, None])
    return dx, (dy * xhat).sum(0), dy.sum(0)


def to_heads(x, b, s, n, d):
    return x.reshape(b, s, n, d).transpose(0, 2, 1, 3)


def from_heads(x):
    b, n, s, d = x.shape
    return x.transpose(0, 2, 1, 3).reshape(b * s, n * d)


def attention(a, w_qkv, b_qkv, w_d, b_d, cfg: RefConfig):
    h, d = cfg.h, cfg.d
    qkv = a @ w_qkv + b_qkv
    q, k, v = (to_heads(qkv[:, i * h:(i + 1) * h], cfg.b, cfg.s, cfg.n, d) for i in range(3))
    probs = softmax_last((q @ k.transpose(0, 1, 3, 2)) / math.sqrt(d))
    ctx = from_heads(probs @ v)
    return ctx @ w_d + b_d, dict(a=a, q=q, k=k, v=v, probs=probs, ctx=ctx, qkv=qkv)


def attention_grad(dout, rec, w_qkv, w_d, cfg: RefConfig):
    d = cfg.d
    g_bd = dout.sum(0)
    g_wd = rec["ctx"].T @ dout
    dheads = to_heads(dout @ w_d.T, cfg.b, cfg.s, cfg.n, d)
    p = rec["probs"]
    dp = dheads @ rec["v"].transpose(0, 1, 3, 2)
    dv = p.transpose(0, 1, 3, 2) @ dheads
    ds = p * (dp - (dp * p).sum(-1, keepdims=True)) / math.sqrt(d)
    dq = ds @ rec["k"]
    dk = ds.transpose(0, 1, 3, 2) @ rec["q"]
    dqkv = np.concatenate([from_heads(dq), from_heads(dk), from_heads(dv)], axis=1)
    return dqkv @ w_qkv.T, rec["a"].T @ dqkv, dqkv.sum(0), g_wd, g_bd


def cross_entropy(logits, labels_flat):
    """Per-token loss log-sum-exp - x_label, and the softmax (layers.py:539-608)."""
    mx = logits.max(-1)
    e = np.exp(logits - mx[:, None])
    z = e.sum(-1)
    picked = logits[np.arange(logits.shape[0]), labels_flat]
    return np.log(z) + mx - picked, e / z[:, None]


# ----------------------------------------------------------------- model

def serial_forward(cfg: RefConfig, params: dict, tokens: np.ndarray, labels: np.ndarray):
    """Mean token cross-entropy loss and the tape needed by serial_backward."""
    if tokens.min() < 0 or tokens.max() >= cfg.v or labels.min() < 0 or labels.max() >= cfg.v:
        raise ValueError("token / label ids out of range")
    x = params["table"][tokens.reshape(-1)]
    tape = []
    for i in range(cfg.num_layers):
        p = f"layers.{i}."
        a1, ln1 = layernorm(x, params[p + "ln1_gamma"], params[p + "ln1_beta"], cfg.eps)
        att, arec = attention(a1, params[p + "w_qkv"], params[p + "b_qkv"], params[p + "w_dense"],
                              params[p + "b_dense"], cfg)
        y1 = x + att
        a2, ln2 = layernorm(y1, params[p + "ln2_gamma"], params[p + "ln2_beta"], cfg.eps)
        mid = a2 @ params[p + "w1"] + params[p + "b1"]
        act = gelu(mid)
        out = y1 + act @ params[p + "w2"] + params[p + "b2"]
        tape.append(dict(x=x, ln1=ln1, a1=a1, attn=arec, att=att, y1=y1, ln2=ln2, a2=a2, mid=mid, act=act,
                         out=out))
        x = out
    logits = x @ params["table"].T
    losses, sm = cross_entropy(logits, labels.reshape(-1))
    loss = float(losses.sum() / (cfg.b * cfg.s))
    return loss, dict(tokens=tokens, labels=labels, layers=tape, x_final=x, logits=logits, softmax=sm,
                      losses=losses, x0=params["table"][tokens.reshape(-1)])


def serial_backward(cfg: RefConfig, params: dict, saved: dict, upstream: float = 1.0) -> dict:
    ntok = cfg.b * cfg.s
    g_logits = saved["softmax"] * (upstream / ntok)
    g_logits[np.arange(ntok), saved["labels"].reshape(-1)] -= upstream / ntok
    grads = {"table": g_logits.T @ saved["x_final"]}
    dx = g_logits @ params["table"]
    grads["_dx_final"] = dx.copy()
    for i in reversed(range(cfg.num_layers)):
        p = f"layers.{i}."
        rec = saved["layers"][i]
        grads[p + "b2"] = dx.sum(0)
        grads[p + "w2"] = rec["act"].T @ dx
        dmid = (dx @ params[p + "w2"].T) * gelu_grad(rec["mid"])
        grads[p + "b1"] = dmid.sum(0)
        grads[p + "w1"] = rec["a2"].T @ dmid
        d_y1, grads[p + "ln2_gamma"], grads[p + "ln2_beta"] = layernorm_grad(dmid @ params[p + "w1"].T,
                                                                             rec["ln2"])
        dy1 = dx + d_y1
        da1, grads[p + "w_qkv"], grads[p + "b_qkv"], grads[p + "w_dense"], grads[p + "b_dense"] = \
            attention_grad(dy1, rec["attn"], params[p + "w_qkv"], params[p + "w_dense"], cfg)
        d_x, grads[p + "ln1_gamma"], grads[p + "ln1_beta"] = layernorm_grad(da1, rec["ln1"])
        dx = dy1 + d_x
    np.add.at(grads["table"], saved["tokens"].reshape(-1), dx)
    grads["_dx0"] = dx
    return grads


def finite_diff(f, arr: np.ndarray, idx, step: float = 1e-4) -> float:
    """Central difference of scalar f() w.r.t. arr[idx] (oracle.py:217-234)."""
    keep = arr[idx]
    arr[idx] = keep + step
    up = f()
    arr[idx] = keep - step
    dn = f()
    arr[idx] = keep
    return (up - dn) / (2 * step)
