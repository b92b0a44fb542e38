"""One BERT-large 1x1 training step after warm-up (ncu target: --steps are counted by the launch filter)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2104_05343_b200 as sg  # noqa: E402


def main():
    layers = int(sys.argv[1]) if len(sys.argv) > 1 else 24
    mesh = sg.create_mesh(sg.MeshConfig(rows=1, cols=1))
    cfg = sg.ModelConfig(b=32, s=512, h=1024, n=16, v=30522, num_layers=layers)
    model = sg.MeshModel(mesh, cfg, None, seed=1)
    ws = model.make_workspace()
    rng = np.random.default_rng(0)
    tok = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).cuda()
    lab = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).cuda()
    for _ in range(2):
        model.train_step(tok, lab, ws, 1e-4)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStart()
    model.train_step(tok, lab, ws, 1e-4)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()


if __name__ == "__main__":
    main()
