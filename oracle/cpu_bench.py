"""Timed CPU baseline of the reference algorithm — TEST / BENCH INFRASTRUCTURE ONLY.

Used by bench.py's ``cpu_baseline`` leg and ``--impl reference`` arm: the
float64 numpy restatement (oracle/model_ref.py, same math as the reference's
serial model and mesh operators) runs a bounded sample of the bench workload
on the host cores, and the measured time is scaled to the full workload:

    t_step(N layers, b) = t_head(b) + N * t_layer(b)     (linear in N, as the
    reference's checkpointed driver is: membuf.py:219-266)

The sample is one transformer layer forward + backward and the embedding /
lm-head / cross-entropy forward + backward at a small batch.
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import model_ref as M


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def _layer_params(cfg: M.RefConfig, rng) -> dict:
    h = cfg.h
    lim = 1.0 / np.sqrt(h)
    p = {"w_qkv": rng.uniform(-lim, lim, (h, 3 * h)), "w_dense": rng.uniform(-lim, lim, (h, h)),
         "w1": rng.uniform(-lim, lim, (h, 4 * h)), "w2": rng.uniform(-lim, lim, (4 * h, h))}
    for k, w in (("b_qkv", 3 * h), ("b_dense", h), ("b1", 4 * h), ("b2", h), ("ln1_beta", h), ("ln2_beta", h)):
        p[k] = np.zeros(w)
    p["ln1_gamma"] = np.ones(h)
    p["ln2_gamma"] = np.ones(h)
    return p


def time_layer(cfg: M.RefConfig, seed: int = 0) -> float:
    """Seconds for one pre-norm layer forward + backward at cfg.b (layers.py:700-759)."""
    rng = np.random.default_rng(seed)
    p = _layer_params(cfg, rng)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    dy = rng.standard_normal(x.shape)
    t0 = time.perf_counter()
    a1, ln1 = M.layernorm(x, p["ln1_gamma"], p["ln1_beta"], cfg.eps)
    att, arec = M.attention(a1, p["w_qkv"], p["b_qkv"], p["w_dense"], p["b_dense"], cfg)
    y1 = x + att
    a2, ln2 = M.layernorm(y1, p["ln2_gamma"], p["ln2_beta"], cfg.eps)
    mid = a2 @ p["w1"] + p["b1"]
    act = M.gelu(mid)
    _ = y1 + act @ p["w2"] + p["b2"]
    _ = act.T @ dy
    dmid = (dy @ p["w2"].T) * M.gelu_grad(mid)
    _ = a2.T @ dmid
    d_y1, _, _ = M.layernorm_grad(dmid @ p["w1"].T, ln2)
    dy1 = dy + d_y1
    da1 = M.attention_grad(dy1, arec, p["w_qkv"], p["w_dense"], cfg)[0]
    M.layernorm_grad(da1, ln1)
    return time.perf_counter() - t0


def time_head(cfg: M.RefConfig, seed: int = 0) -> float:
    """Seconds for embedding + tied lm-head + mean cross entropy, forward + backward."""
    rng = np.random.default_rng(seed)
    table = rng.uniform(-1 / np.sqrt(cfg.h), 1 / np.sqrt(cfg.h), (cfg.v, cfg.h))
    tokens = rng.integers(0, cfg.v, (cfg.b, cfg.s)).reshape(-1)
    labels = rng.integers(0, cfg.v, (cfg.b, cfg.s)).reshape(-1)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    t0 = time.perf_counter()
    _ = table[tokens]
    logits = x @ table.T
    losses, sm = M.cross_entropy(logits, labels)
    g = sm / losses.size
    g[np.arange(losses.size), labels] -= 1.0 / losses.size
    _ = g @ table
    tg = g.T @ x
    np.add.at(tg, tokens, x)
    return time.perf_counter() - t0


def training_samples_per_sec(h: int, n: int, s: int, v: int, layers: int, b_sample: int = 2) -> dict:
    """Extrapolated CPU training throughput of the full stack from a bounded sample."""
    cfg = M.RefConfig(b=b_sample, s=s, h=h, n=n, v=v, num_layers=1)
    t_layer = time_layer(cfg)
    t_head = time_head(cfg)
    t_step = t_head + layers * t_layer
    return {"samples_per_s": b_sample / t_step, "t_layer_s": t_layer, "t_head_s": t_head,
            "sample": f"oracle fp64 fwd+bwd of 1 layer + embedding/lm-head/CE at b={b_sample}, s={s}, h={h}, "
                      f"n={n}, v={v}; step time = head + {layers} x layer (extrapolated)"}


def time_layer_forward(cfg: M.RefConfig, seed: int = 0) -> float:
    """Seconds for one pre-norm layer forward at cfg.b (layers.py:700-725)."""
    rng = np.random.default_rng(seed)
    p = _layer_params(cfg, rng)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    t0 = time.perf_counter()
    a1, _ = M.layernorm(x, p["ln1_gamma"], p["ln1_beta"], cfg.eps)
    att, _ = M.attention(a1, p["w_qkv"], p["b_qkv"], p["w_dense"], p["b_dense"], cfg)
    y1 = x + att
    a2, _ = M.layernorm(y1, p["ln2_gamma"], p["ln2_beta"], cfg.eps)
    _ = y1 + M.gelu(a2 @ p["w1"] + p["b1"]) @ p["w2"] + p["b2"]
    return time.perf_counter() - t0


def time_head_forward(cfg: M.RefConfig, seed: int = 0) -> float:
    """Seconds for embedding + tied lm-head + mean cross entropy, forward only."""
    rng = np.random.default_rng(seed)
    table = rng.uniform(-1 / np.sqrt(cfg.h), 1 / np.sqrt(cfg.h), (cfg.v, cfg.h))
    tokens = rng.integers(0, cfg.v, (cfg.b, cfg.s)).reshape(-1)
    labels = rng.integers(0, cfg.v, (cfg.b, cfg.s)).reshape(-1)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h))
    t0 = time.perf_counter()
    _ = table[tokens]
    M.cross_entropy(x @ table.T, labels)
    return time.perf_counter() - t0


def inference_samples_per_sec(h: int, n: int, s: int, v: int, layers: int, b_sample: int = 1) -> dict:
    """Extrapolated CPU forward (inference) throughput of the full stack from a bounded sample."""
    cfg = M.RefConfig(b=b_sample, s=s, h=h, n=n, v=v, num_layers=1)
    t_layer = time_layer_forward(cfg)
    t_head = time_head_forward(cfg)
    t_step = t_head + layers * t_layer
    return {"samples_per_s": b_sample / t_step, "t_layer_s": t_layer, "t_head_s": t_head,
            "sample": f"oracle fp64 forward of 1 layer + embedding/lm-head/CE at b={b_sample}, s={s}, h={h}, "
                      f"n={n}, v={v}; forward time = head + {layers} x layer (extrapolated)"}


def summa_tflops(n: int = 4096) -> dict:
    """fp64 numpy product at N^3 (the reference's local_matmul, mesh.py:354-361)."""
    rng = np.random.default_rng(0)
    a, b = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    t0 = time.perf_counter()
    _ = a @ b
    dt = time.perf_counter() - t0
    return {"tflops": 2.0 * n ** 3 / dt / 1e12, "seconds": dt, "n": n}
