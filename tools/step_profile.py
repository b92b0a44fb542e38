"""Per-kernel breakdown of one training step (torch.profiler / CUPTI) plus the
per-shape GEMM table from CUDA events. Usage: python tools/step_profile.py [--layers L]"""
import argparse
import collections
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2104_05343_b200 as sg  # noqa: E402
from paper_2104_05343_b200 import kernels as K  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=24)
    ap.add_argument("--b", type=int, default=32)
    ap.add_argument("--rows", type=int, default=1)
    ap.add_argument("--cols", type=int, default=1)
    args = ap.parse_args()
    mesh = sg.create_mesh(sg.MeshConfig(rows=args.rows, cols=args.cols))
    cfg = sg.ModelConfig(b=args.b, s=512, h=1024, n=16, v=30522, num_layers=args.layers)
    model = sg.MeshModel(mesh, cfg, None, seed=1)
    ws = model.make_workspace()
    rng = np.random.default_rng(0)
    tok = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).cuda()
    lab = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).cuda()
    for _ in range(3):
        model.train_step(tok, lab, ws, 1e-4)
    torch.cuda.synchronize()
    with K.profile_gemms() as prof:
        model.train_step(tok, lab, ws, 1e-4)
    torch.cuda.synchronize()
    by = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for fl, e0, e1, shape in prof.records:
        d = by[shape]
        d[0] += 1
        d[1] += e0.elapsed_time(e1)
        d[2] += fl
    print("GEMM shapes (M, N, K, batch): count, ms, TFLOP/s")
    for shape, (n, ms, fl) in sorted(by.items(), key=lambda kv: -kv[1][1]):
        print(f"  {shape}: {n:4d} {ms:8.3f} ms {fl / ms / 1e9:8.1f}")
    print("total", prof.summary())
    from torch.profiler import ProfilerActivity, profile

    with profile(activities=[ProfilerActivity.CUDA]) as p:
        model.train_step(tok, lab, ws, 1e-4)
        torch.cuda.synchronize()
    agg = collections.defaultdict(lambda: [0, 0.0])
    for ev in p.events():
        if ev.device_type == torch.autograd.DeviceType.CUDA:
            name = ev.name[:90]
            agg[name][0] += 1
            agg[name][1] += ev.device_time_total / 1e3 if hasattr(ev, "device_time_total") else ev.cuda_time_total / 1e3
    tot = sum(v[1] for v in agg.values())
    print(f"all kernels: {tot:.2f} ms")
    for name, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:30]:
        print(f"  {ms:8.3f} ms {100 * ms / tot:5.1f}% x{n:5d}  {name}")


if __name__ == "__main__":
    main()
