"""Large square products under different rasterisation group heights (SG_GEMM_GROUP_M), each in a subprocess."""
import os
import subprocess
import sys

code = r'''
import sys, torch
sys.path.insert(0, ".")
from paper_2104_05343_b200 import kernels as K
from tools.gemm_step_shapes import bench
for N in (8192, 16384, 32768):
    a = torch.randn(N, N, device="cuda").bfloat16(); b = torch.randn(N, N, device="cuda").bfloat16(); o = torch.empty(N, N, device="cuda").bfloat16()
    us = bench(lambda: K.gemm(a, b, o), iters=5 if N < 32768 else 2, warm=2)
    print(f"group={sys.argv[1]} N={N}: {us/1e3:.2f} ms {2.0*N**3/us/1e6:.0f} TF/s", flush=True)
    del a, b, o
'''
for g in sys.argv[1:] or ["16", "4", "8", "32", "64"]:
    env = dict(os.environ, SG_GEMM_GROUP_M=g)
    subprocess.run([sys.executable, "-c", code, g], env=env)
