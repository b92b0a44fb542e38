"""Weight-gradient (fused SGD, D += -lr A^T B in place) timings under forced split-K counts (SG_GEMM_SPLITS)."""
import os, subprocess, sys
code = r'''
import os, sys, torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K
from tools.gemm_step_shapes import bench
M, h = 16384, 1024
r = lambda *s: torch.randn(*s, device="cuda").bfloat16()
x, dmid, dy, act, dqkv = r(M, h), r(M, 4*h), r(M, h), r(M, 4*h), r(M, 3*h)
g1 = torch.zeros(h, 4*h, device="cuda"); g2 = torch.zeros(4*h, h, device="cuda"); gq = torch.zeros(h, 3*h, device="cuda")
for name, a, b, o in [("dW1", x.t(), dmid, g1), ("dW2", act.t(), dy, g2), ("dWqkv", x.t(), dqkv, gq)]:
    us = bench(lambda: K.gemm(a, b, o, c=o, alpha=-1e-4))
    print(f"{name} splits={os.environ.get('SG_GEMM_SPLITS','auto')}: {us:.1f} us {2*a.shape[0]*a.shape[1]*b.shape[1]/us/1e6:.0f} TF/s", flush=True)
'''
for s in ["", "2", "3", "4", "5", "7", "8"]:
    env = dict(os.environ)
    if s: env["SG_GEMM_SPLITS"] = s
    subprocess.run([sys.executable, "-c", code], env=env)
