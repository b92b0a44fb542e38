"""NVLink bandwidth probe for the SUMMA roofline's panel term.

Measures, between GPU 0 and every other visible GPU, the per-direction bandwidth of
copy-engine peer copies (a device-to-device torch copy across GPUs) of a panel-sized
buffer, with CUDA events. Writes profiles/nvlink_probe.json
(``gbs`` = the median peer-copy bandwidth), which bench.py's per-GEMM roofline reads
instead of the 900 GB/s NVLink 5 figure. With one visible GPU it records why nothing
was measured.

    python tools/nvlink_probe.py [--mib 256]
"""

from __future__ import annotations

import argparse
import json
import statistics
from pathlib import Path

import torch

OUT = Path(__file__).resolve().parents[1] / "profiles" / "nvlink_probe.json"


def _time(fn, iters=10) -> float:
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / iters * 1e-3


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    args = ap.parse_args()
    n = torch.cuda.device_count()
    res = {"gpus": n, "bytes": args.mib << 20}
    if n < 2:
        res.update({"gbs": None, "unavailable": f"{n} visible GPU: no peer link to measure"})
    else:
        src = torch.empty(args.mib << 20, dtype=torch.uint8, device="cuda:0")
        pairs = {}
        for d in range(1, n):
            dst = torch.empty_like(src, device=f"cuda:{d}")
            with torch.cuda.device(0):
                t = _time(lambda: dst.copy_(src, non_blocking=True))
            pairs[f"0->{d}"] = src.numel() / t / 1e9
        res["peer_copy_gbs"] = pairs
        res["gbs"] = statistics.median(pairs.values())
    OUT.write_text(json.dumps(res, indent=1) + "\n")
    print(json.dumps(res))


if __name__ == "__main__":
    main()
