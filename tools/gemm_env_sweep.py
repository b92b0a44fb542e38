"""Step GEMM shapes under the sg_gemm tuning overrides (SG_GEMM_BN / _PAIR /
_EPI_WARPS are read once per process, so every variant runs in a subprocess).

    python tools/gemm_env_sweep.py            # all cases x all variants
    python tools/gemm_env_sweep.py --one CASE  # (child) time one case
"""
import os
import subprocess
import sys

VARIANTS = [
    {},
]
_ALL_VARIANTS = [
    {},
    {"SG_GEMM_BN": "128"},
    {"SG_GEMM_EPI_WARPS": "4"},
    {"SG_GEMM_EPI_WARPS": "8"},
    {"SG_GEMM_PAIR": "0"},
]
CASES = ["qkv", "dense", "fc1", "fc2", "dctx", "dWd", "dWqkv", "dW1", "dW2", "dmid", "dxln"]


def child(case):
    import torch

    sys.path.insert(0, ".")
    from paper_2104_05343_b200 import kernels as K

    M, h = 16384, 1024
    bf = torch.bfloat16
    r = lambda *s: torch.randn(*s, device="cuda").to(bf)  # noqa: E731
    if case == "qkv":
        a, b, o, kw = r(M, h), r(h, 3 * h), torch.empty(M, 3 * h, device="cuda", dtype=bf), {
            "bias": torch.randn(3 * h, device="cuda")}
    elif case == "dense":
        a, b, o = r(M, h), r(h, h), torch.empty(M, h, device="cuda")
        kw = {"bias": torch.randn(h, device="cuda"), "c": torch.randn(M, h, device="cuda")}
    elif case == "fc1":
        a, b, o = r(M, h), r(h, 4 * h), torch.empty(M, 4 * h, device="cuda", dtype=bf)
        kw = {"bias": torch.randn(4 * h, device="cuda"), "act": K.ACT_GELU, "aux": torch.empty_like(o)}
    elif case == "fc2":
        a, b, o = r(M, 4 * h), r(4 * h, h), torch.empty(M, h, device="cuda")
        kw = {"bias": torch.randn(h, device="cuda"), "c": torch.randn(M, h, device="cuda")}
    elif case == "dmid":  # dy W2^T with GELU' from the saved pre-activation
        a, b, o = r(M, h), r(4 * h, h).t(), torch.empty(M, 4 * h, device="cuda", dtype=bf)
        kw = {"act": K.ACT_DGELU, "aux": r(M, 4 * h), "colsum": torch.zeros(4 * h, device="cuda")}
    elif case == "dxln":  # dmid W1^T with the LayerNorm-backward statistics
        a, b, o = r(M, 4 * h), r(h, 4 * h).t(), torch.empty(M, h, device="cuda")
        x = torch.randn(M, h, device="cuda")
        kw = {"ln_stats": (x, torch.randn(h, device="cuda"), x.mean(1), torch.ones(M, device="cuda"),
                           torch.zeros(M, 2, device="cuda"))}
    elif case == "dctx":
        a, b, o, kw = r(M, h), r(h, h).t(), torch.empty(M, h, device="cuda", dtype=bf), {}
    elif case == "dWd":
        a, b, o, kw = r(M, h).t(), r(M, h), torch.empty(h, h, device="cuda"), {}
    elif case == "dW1":
        a, b, o, kw = r(M, h).t(), r(M, 4 * h), torch.empty(h, 4 * h, device="cuda"), {}
    elif case == "dW2":
        a, b, o, kw = r(M, 4 * h).t(), r(M, h), torch.empty(4 * h, h, device="cuda"), {}
    elif case == "dWqkv":
        a, b, o, kw = r(M, h).t(), r(M, 3 * h), torch.empty(h, 3 * h, device="cuda"), {}
    else:
        raise SystemExit(case)
    fl = 2.0 * a.shape[0] * a.shape[1] * b.shape[1]
    fn = lambda: K.gemm(a, b, o, **kw)  # noqa: E731
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    n = 30
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
    print(f"{us:.1f} {fl / us / 1e6:.0f}")


def main():
    if len(sys.argv) > 2 and sys.argv[1] == "--one":
        return child(sys.argv[2])
    global VARIANTS
    args = sys.argv[1:]
    if args and args[0] == "--all":
        VARIANTS, args = _ALL_VARIANTS, args[1:]
    cases = args or CASES
    for case in cases:
        row = []
        for v in VARIANTS:
            env = dict(os.environ, **v)
            out = subprocess.run([sys.executable, __file__, "--one", case], env=env, capture_output=True, text=True)
            res = out.stdout.strip().splitlines()[-1] if out.returncode == 0 and out.stdout.strip() else "ERR"
            row.append(f"{'+'.join(f'{k[8:]}={x}' for k, x in v.items()) or 'default'}: {res}")
        print(f"{case:6s} | " + " | ".join(row), flush=True)


if __name__ == "__main__":
    main()
