#!/usr/bin/env python
"""Bench: 2D (SUMMA) transformer training throughput on B200 — BASELINE.json's metric
"2D transformer train samples/sec & SUMMA TFLOP/s at 1/2/4/8 B200 vs CPU ref".

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (one process per GPU)

Workload (configs[2]): BERT-large-shaped 2D stack — 24 pre-norm layers, h=1024,
16 heads, s=512, global batch 32, BERT vocabulary 30522 with the tied lm-head
and cross entropy — trained with SGD on an r x c mesh (1 -> 1x1, 2 -> 1x2,
4 -> 2x2, 8 -> 2x4), global batch fixed ("strong"). Synthetic random-init
weights and uniform random token / label ids (no datasets offline).

value : samples/s with inputs resident in HBM, K steps between barrier +
        synchronize, CUDA events, max over ranks.
e2e   : same metric through the public API (MeshModel.train_step) with the
        tokens / labels copied from pinned host memory and the loss read back
        every step.
summa : SUMMA AB / AB^T / A^T B TFLOP/s at N=8192 bf16 on the same mesh (configs[1]).
roofline : tcgen05 GEMM kernel, algorithmic FLOPs / CUDA-event time of every
        launch of one instrumented step, vs measured cuBLAS sustained peak.
cpu_baseline : the float64 oracle restatement of the reference on the host
        cores, bounded sample (oracle/cpu_bench.py), rank 0 at N = 1.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
# the CPU legs (cpu_baseline, --impl reference) use every host core; OpenBLAS reads this
# when numpy is first imported, so it is set before anything imports numpy
os.environ.setdefault("OPENBLAS_NUM_THREADS", str(len(os.sched_getaffinity(0))))

METRIC = "2D transformer train samples/sec & SUMMA TFLOP/s at 1/2/4/8 B200 vs CPU ref"
WORKLOADS = {
    "bert": dict(b=32, s=512, h=1024, n=16, v=30522, layers=24, name="bert-large-2d-stack-train"),
    "gpt": dict(b=8, s=2048, h=4096, n=32, v=50257, layers=24, name="gpt-h4096-2d-stack-train"),
}


def parse():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawDescriptionHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--workload", choices=tuple(WORKLOADS), default="bert")
    ap.add_argument("--batch", type=int, default=0, help="override the global batch")
    ap.add_argument("--layers", type=int, default=0, help="override the layer count")
    ap.add_argument("--no-graph", action="store_true", help="do not capture the step into a CUDA graph")
    ap.add_argument("--checkpointing", action="store_true", help="activation checkpointing (recompute)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--summa-n", type=int, default=8192)
    ap.add_argument("--summa-sweep", action="store_true",
                    help="also time the SUMMA forms at N = 4096, 8192, 16384, 32768 (configs[1])")
    ap.add_argument("--mode", choices=("train", "infer"), default="train",
                    help="train: fwd+bwd+SGD step; infer: forward (with the CE loss, as the reference) only")
    ap.add_argument("--max-batch", action="store_true",
                    help="after the timed run, find the largest global batch that fits (doubling, then bisection)")
    ap.add_argument("--placement", choices=("natural", "bunched"), default="natural",
                    help="rank placement of the mesh positions (mesh.py:230-275)")
    ap.add_argument("--node-size", type=int, default=0,
                    help="GPUs per placement node (default: all GPUs of the run = one NVSwitch node)")
    ap.add_argument("--compare-1d", choices=("auto", "on", "off"), default="auto",
                    help="also time one 2D layer against the Megatron 1D layer on the same GPUs (auto: N > 1)")
    return ap.parse_args()


def workload(args) -> dict:
    w = dict(WORKLOADS[args.workload])
    if args.mode == "infer":
        w["name"] = w["name"].replace("-train", "-infer")
    if args.batch:
        w["b"] = args.batch
    if args.layers:
        w["layers"] = args.layers
    return w


def model_flops(w: dict, mode: str = "train") -> float:
    """Algorithmic FLOPs of one fwd+bwd step (costmodel.py:63-65 x3, + lm-head 2bsvh x3), or of
    the forward alone in inference mode."""
    b, s, h, v, L = w["b"], w["s"], w["h"], w["v"], w["layers"]
    per_layer_fwd = 2.0 * (12 * b * s * h * h + 2 * b * s * s * h)
    return (1.0 if mode == "infer" else 3.0) * (L * per_layer_fwd + 2.0 * b * s * v * h)


def cpu_sample(w: dict, mode: str) -> dict:
    """One bounded CPU sample of the workload: one layer (+ embedding / lm-head / CE) at the
    bench's own batch for the BERT shape (~6 fp64 TFLOP, 10-20 s on the box's host cores),
    at b = 1 for the h = 4096 stack (one such layer at b = 8 is ~20 fp64 TFLOP)."""
    from oracle import cpu_bench

    b_sample = w["b"] if w["h"] <= 1024 else 1
    if mode == "infer":
        return cpu_bench.inference_samples_per_sec(w["h"], w["n"], w["s"], w["v"], w["layers"], b_sample=b_sample)
    return cpu_bench.training_samples_per_sec(w["h"], w["n"], w["s"], w["v"], w["layers"], b_sample=b_sample)


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"bf16_burst": d.get("bf16_tflops", 1590.0), "bf16_sustained": d.get("bf16_tflops_sustained", 1409.0),
                "hbm": d.get("hbm_gbs", 6650.0), "src": "measured (MEASURED_PEAKS.json)"}
    return {"bf16_burst": 1590.0, "bf16_sustained": 1400.0, "hbm": 6650.0, "src": "fallback (B200_PROFILING.md)"}


_FORM = {"qkv": "ab", "dense": "ab", "fc1": "ab", "fc2": "ab", "dx_lmhead": "ab", "dctx": "abt", "dact": "abt",
         "dx_qkv": "abt", "dx_fc1": "abt", "logits": "abt", "dw_dense": "atb", "dw_qkv": "atb", "dw1": "atb",
         "dw2": "atb", "dw_table": "atb"}


def nvlink_peak() -> dict:
    """Per-direction NVLink bandwidth: tools/nvlink_probe.py's measurement when committed,
    else the B200 NVLink 5 figure (900 GB/s per direction)."""
    p = ROOT / "profiles" / "nvlink_probe.json"
    if p.exists():
        d = json.loads(p.read_text())
        if d.get("gbs"):
            return {"gbs": d["gbs"], "src": "measured (profiles/nvlink_probe.json)"}
    return {"gbs": 900.0, "src": "spec (NVLink 5, per direction; unmeasured: one-GPU pool)"}


def gemm_rooflines(by_tag: dict, mesh, pk: dict) -> list:
    """Each SUMMA product of the step against its roofline: the slower of the tensor-core
    time (2 M N K / sustained bf16 peak) and its panel bytes per device at NVLink bandwidth
    (SURVEY.md §8d). Per local launch (M, N, K): AB receives the A panel M K (all but the
    root column's steps) and the B panel K N (all but the root row's); AB^T receives the
    B^T panel N K and sends its fp32 partial M N to the row destination; A^T B receives the
    A panel K M and sends its fp32 partial M N to the column destination."""
    r, c = mesh.r, mesh.c
    fa, fb = (c - 1) / c, (r - 1) / r
    nv = nvlink_peak()
    rows = []
    for tag, d in sorted(by_tag.items(), key=lambda kv: -kv[1]["ms"]):
        form = _FORM.get(tag)
        panel = 0.0
        for (M, N, K, batch), count in d["shapes"].items():
            per = {"ab": 2 * M * K * fa + 2 * K * N * fb, "abt": 2 * N * K * fb + 4 * M * N * fa,
                   "atb": 2 * K * M * fa + 4 * M * N * fb}.get(form, 0.0) * batch
            panel += per * count
        t_tensor = d["flops"] / (pk["bf16_sustained"] * 1e12) * 1e3
        t_link = panel / (nv["gbs"] * 1e9) * 1e3
        roof = max(t_tensor, t_link)
        rows.append({"product": tag, "form": form, "launches": d["launches"], "ms": d["ms"],
                     "tflops": d["flops"] / (d["ms"] * 1e-3) / 1e12 if d["ms"] > 0 else None,
                     "roofline_ms": roof, "bound": "nvlink" if t_link > t_tensor else "tensor",
                     "frac": roof / d["ms"] if d["ms"] > 0 else None, "panel_bytes": panel,
                     "local_shapes": {"x".join(map(str, k)): v for k, v in d["shapes"].items()}})
    if rows:
        rows[0]["peaks"] = {"tensor": f"{pk['bf16_sustained']} TF/s ({pk['src']} sustained)",
                            "nvlink": f"{nv['gbs']} GB/s ({nv['src']})"}
    return rows


def gemm_traffic():
    """DRAM bytes per GEMM launch of one training step from the newest committed ncu
    capture (profiles/*_gemm_traffic.json, written by tools/summarize_ncu.py)."""
    files = sorted((ROOT / "profiles").glob("*_gemm_traffic.json"), key=lambda p: p.stat().st_mtime)
    if not files:
        return None
    d = json.loads(files[-1].read_text())
    d["file"] = f"profiles/{files[-1].name}"
    return d


# ----------------------------------------------------------------------------- clocks

class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.idx = gpu_index
        self.proc = None
        self.out = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                                          "-i", str(self.idx), "-lms", "200"], stdout=self.out,
                                         stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        self.out.flush()
        rows = []
        for line in Path(self.out.name).read_text().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) >= 9 and parts[1].isdigit():
                rows.append(parts)
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        reasons = sorted({n for r in rows for n, v in zip(names, r[5:9]) if v.lower().startswith("active")})
        return {"sm_mhz": statistics.median(float(r[1]) for r in rows), "sm_max_mhz": float(rows[0][2]),
                "reasons": reasons, "samples": len(rows),
                "power_w_max": max(float(r[3]) for r in rows if r[3].replace(".", "").isdigit()) if rows else None}


# ----------------------------------------------------------------------------- reference arm

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import cpu_bench

    w = workload(args)
    cores = cpu_bench.host_cores()
    vals, walls = [], []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        r = cpu_sample(w, args.mode)
        if i >= args.warmup:
            vals.append(r["samples_per_s"])
            walls.append(time.perf_counter() - t0)
    v = statistics.mean(vals)
    # a "step" of this arm is the bounded sample (one layer + embedding / lm-head / CE):
    # ms_per_step is its measured wall time, value the full stack's throughput derived
    # from it (step time = head + layers x layer, the reference's cost is linear in layers)
    line = {"metric": METRIC, "impl": "reference", "value": v, "unit": "samples/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": statistics.mean(walls) * 1e3,
            "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": _config(w, args.gpus, args, extra={
                "note": "reference CPU algorithm (numpy f64 oracle port); each step is a bounded sample "
                        "(one layer + embedding / lm-head / CE); value = the full stack's samples/s "
                        f"(full-stack step {w['b'] / v:.1f} s, extrapolated)"}),
            "cpu_baseline": {"value": v, "unit": "samples/s", "cores": cores, "kind": "port", "sample": r["sample"]},
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(w, n_gpus, args, extra=None) -> dict:
    from paper_2104_05343_b200.mesh import mesh_for_world

    mc = mesh_for_world(n_gpus)
    cfg = {"workload": w["name"], "placement": args.placement, "model": f"2D transformer L={w['layers']} h={w['h']} n={w['n']} v={w['v']}",
           "global_batch": w["b"], "seq_len": w["s"], "hidden": w["h"], "heads": w["n"], "layers": w["layers"],
           "vocab": w["v"], "mesh": f"{mc.rows}x{mc.cols}", "parallelism": f"2d-summa r{mc.rows}xc{mc.cols}",
           "checkpointing": bool(args.checkpointing), "cuda_graph": not args.no_graph,
           "mode": args.mode, "optimizer": "sgd" if args.mode == "train" else None, "l2": "working set (weights fp32+bf16, >10 GB activations) larger than the 126 MB L2"}
    if extra:
        cfg.update(extra)
    return cfg


# ----------------------------------------------------------------------------- our arm

def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
        return
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2104_05343_b200 as sg
    from paper_2104_05343_b200 import kernels as K

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        if world == 1 and args.gpus > 1:
            raise SystemExit("--gpus N > 1 must be launched with torchrun (one process per GPU)")
    torch.cuda.set_device(local)
    if world > 1:
        # NCCL's panel broadcasts run beside the persistent GEMMs, which leave SG_SM_RESERVE
        # SMs free (mesh.py); cap NCCL's channels (one CTA each) to that budget
        os.environ.setdefault("NCCL_MAX_NCHANNELS", os.environ.get("SG_SM_RESERVE", "8"))
        sg.init_dist("nccl", device_id=torch.device("cuda", local))  # async NCCL errors + collective timeout
    w = workload(args)
    mc = sg.mesh_for_world(world)
    mc = sg.MeshConfig(rows=mc.rows, cols=mc.cols, node_size=args.node_size or world,
                       placement=sg.Placement(args.placement))
    mesh = sg.create_mesh(mc, backend="dist" if world > 1 else "local")
    cfg = sg.ModelConfig(b=w["b"], s=w["s"], h=w["h"], n=w["n"], v=w["v"], num_layers=w["layers"])
    model = sg.MeshModel(mesh, cfg, None, seed=1234)
    ws = model.make_workspace(checkpointing=args.checkpointing)
    rng = np.random.default_rng(0)
    tok_h = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).pin_memory()
    lab_h = torch.from_numpy(rng.integers(0, cfg.v, (cfg.b, cfg.s))).pin_memory()
    tok_d, lab_d = tok_h.cuda(), lab_h.cuda()
    lr = 1e-4

    def step():
        if args.mode == "infer":
            return model.infer(tok_d, lab_d, ws)
        return model.train_step(tok_d, lab_d, ws, lr, checkpointing=args.checkpointing)

    def barrier():
        if world > 1:
            dist.barrier()

    for _ in range(args.warmup):
        loss = step()
    torch.cuda.synchronize()
    if getattr(mesh, "peer", None) is not None:
        mesh.peer.check()
    use_graph = not args.no_graph
    graph = None
    graph_error = None
    if use_graph:
        # one graph replay per step on every rank: the dist step's NCCL panel broadcasts /
        # statistics all-reduces are captured with it, the peer-memory reduces are plain
        # kernels (device-side barrier epochs, peer.py)
        try:
            s = torch.cuda.Stream()
            s.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(s):
                step()
            torch.cuda.current_stream().wait_stream(s)
            torch.cuda.synchronize()
            barrier()
            graph = torch.cuda.CUDAGraph()
            with torch.cuda.graph(graph):
                loss = step()
            graph.replay()
            torch.cuda.synchronize()
            barrier()
        except Exception as e:  # capture unsupported here: time the eager step instead
            graph, use_graph, graph_error = None, False, f"{type(e).__name__}: {e}"[:300]
            torch.cuda.synchronize()
    if use_graph:
        run = graph.replay
    else:
        def run():
            nonlocal loss
            loss = step()

    # ------------------------------------------------------------- timed region (device-resident inputs)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    launches0 = K.launch_count()
    with ClockSampler(local) as clocks:
        barrier()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            run()
        ev1.record()
        torch.cuda.synchronize()
        barrier()
    launches = K.launch_count() - launches0
    if use_graph:  # replays do not pass through the host wrappers: count one captured step
        l0 = K.launch_count()
        step()
        torch.cuda.synchronize()
        launches = (K.launch_count() - l0) * args.steps
    ms = ev0.elapsed_time(ev1)
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = cfg.b * args.steps / (ms * 1e-3)
    final_loss = float(loss.item())

    # ------------------------------------------------------------- end to end (host buffers)
    h2d = (tok_h.numel() * tok_h.element_size() + lab_h.numel() * lab_h.element_size()) * world
    d2h = 4 * world
    barrier()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        tok_d.copy_(tok_h, non_blocking=True)
        lab_d.copy_(lab_h, non_blocking=True)
        run()
        _ = float(loss.item())  # D2H of the step's loss
    e1.record()
    torch.cuda.synchronize()
    e2e_ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([e2e_ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = cfg.b * args.steps / (e2e_ms * 1e-3)

    # ------------------------------------------------------------- roofline of the dominant kernel
    torch.cuda.synchronize()
    s_ev0, s_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with K.profile_gemms() as prof:
        s_ev0.record()
        step()
        s_ev1.record()
    torch.cuda.synchronize()
    gsum = prof.summary()
    inst_step_ms = s_ev0.elapsed_time(s_ev1)
    pk = peaks()
    per_gemm = gemm_rooflines(prof.by_tag(), mesh, pk)
    traffic = gemm_traffic()
    roof = {"kernel": "sg_gemm (tcgen05 persistent GEMM)", "bound": "tensor", "achieved": gsum["tflops"],
            "peak": pk["bf16_sustained"], "unit": "TFLOP/s", "frac": gsum["tflops"] / pk["bf16_sustained"],
            "traffic": None if traffic is None else traffic["traffic_bytes_per_launch"],
            "traffic_source": None if traffic is None else traffic["file"],
            "peak_source": pk["src"] + " sustained bf16",
            "launches_per_step": gsum["launches"], "gemm_ms_per_step": gsum["ms"],
            # share of the (graph-replayed) step: the instrumented step itself runs eagerly
            # and is host-launch bound, so it is not the denominator
            "gemm_share_of_step": gsum["ms"] / ms_step if ms_step > 0 else None,
            "instrumented_step_ms": inst_step_ms,
            "algorithmic_flops_per_step": gsum["flops"], "per_gemm": per_gemm}

    # ------------------------------------------------------------- SUMMA sweep point (configs[1])
    summa = summa_point(sg, K, mesh, args.summa_n, pk, barrier, world)
    if args.summa_sweep:
        summa["sweep"] = [summa_point(sg, K, mesh, n, pk, barrier, world) for n in (4096, 8192, 16384, 32768)]

    # ------------------------------------------------------------- CPU baseline (rank 0, N = 1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import cpu_bench

        r = cpu_sample(w, args.mode)
        cpu = {"value": r["samples_per_s"], "unit": "samples/s", "cores": cpu_bench.host_cores(), "kind": "port",
               "sample": r["sample"]}

    cmp1d = None
    if args.compare_1d == "on" or (args.compare_1d == "auto" and world > 1):
        cmp1d = compare_1d(sg, K, mesh, w, barrier, world)

    maxb = None
    if args.max_batch:
        import gc

        # free the timed model (and the captured graph's pool) before probing
        run = step = graph = model = ws = None
        gc.collect()
        torch.cuda.empty_cache()
        maxb = max_batch_sweep(sg, mesh, w, args, world)
    if rank == 0:
        flops = model_flops(w, args.mode)
        line = {"metric": METRIC, "value": value, "unit": "samples/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
                "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init weights, uniform token ids)",
                "config": _config(w, world, args, extra={"cuda_graph": use_graph, "graph_error": graph_error,
                                                         "peer_memory": getattr(mesh, "peer", None) is not None,
                                                         "gemm_sm_budget": K.gemm_sm_budget()}),
                "model_tflops": flops / (ms_step * 1e-3) / 1e12,
                "e2e": {"value": e2e_value, "unit": "samples/s", "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h},
                "gpu_launches": int(launches), "roofline": roof, "summa": summa, "cpu_baseline": cpu,
                "clocks": clocks.summary(), "final_loss": final_loss}
        if maxb is not None:
            line["max_batch"] = maxb
        if cmp1d is not None:
            line["optimus_vs_megatron"] = cmp1d
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def compare_1d(sg, K, mesh, w, barrier, world, iters: int = 5) -> dict:
    """One transformer layer fwd + bwd in the 2D (SUMMA) partition against the paper's
    Megatron 1D baseline (baseline.py:40-224) on the same GPUs, same
    shape and parameters: per-layer ms (CUDA events, max over ranks) and the speed-up."""
    import numpy as np
    import torch

    from paper_2104_05343_b200.baseline1d import Baseline1DLayer
    from paper_2104_05343_b200.layers import LayerParams, RowHostedVector, TransformerLayer, interleave_qkv
    from paper_2104_05343_b200.summa import as_bf16

    cfg = sg.ModelConfig(b=w["b"], s=w["s"], h=w["h"], n=w["n"], v=w["v"], num_layers=1)
    g = {k[len("layers.0."):]: v for k, v in sg.init_global_params(cfg, 5).items() if k.startswith("layers.0.")}
    c = mesh.c
    mats = {k: sg.scatter(interleave_qkv(g[k], c) if k == "w_qkv" else g[k], mesh, layout="weight")
            for k in ("w_qkv", "w_dense", "w1", "w2")}
    for m in mats.values():
        m.bf16_twin = as_bf16(m)
    vecs = {k: RowHostedVector.split(interleave_qkv(g[k], c) if k == "b_qkv" else g[k], c, mesh=mesh)
            for k in ("b_qkv", "b_dense", "b1", "b2", "ln1_gamma", "ln1_beta", "ln2_gamma", "ln2_beta")}
    layer2d = TransformerLayer(mesh, cfg, LayerParams(**mats, **vecs))
    layer1d = Baseline1DLayer(mesh, cfg, g)
    rng = np.random.default_rng(1)
    x = rng.standard_normal((cfg.b * cfg.s, cfg.h)).astype(np.float32)
    xs, dys = sg.scatter(x, mesh), sg.scatter(x, mesh)
    xd = torch.as_tensor(x).cuda()

    def run2d():
        ws = sg.Workspace(mesh.p)
        out, saved = layer2d.forward(xs, ws)
        layer2d.backward(dys, saved, ws)

    def run1d():
        ws = sg.Workspace(mesh.p)
        out, saved = layer1d.forward(xd, ws)
        layer1d.backward(xd, saved, ws, host_grads=False)

    res = {"mesh_2d": f"{mesh.r}x{mesh.c}", "partition_1d": f"1x{mesh.p} (Megatron)", "layer": "1 layer fwd+bwd",
           "shape": {k: w[k] for k in ("b", "s", "h", "n")}}
    for name, fn in (("ms_2d", run2d), ("ms_1d", run1d)):
        fn()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        res[name] = ms
    res["speedup_2d_over_1d"] = res["ms_1d"] / res["ms_2d"]
    return res


def max_batch_sweep(sg, mesh, w, args, world) -> dict:
    """Largest global batch whose step (train or infer) runs without running out of HBM:
    double from the bench batch, then bisect. Same mesh and
    model size; a fresh random-init model per probe."""
    import gc

    import numpy as np
    import torch

    r = mesh.r

    def fits(b: int) -> bool:
        model = ws = tok = lab = None
        ok = True
        try:
            cfg = sg.ModelConfig(b=b, s=w["s"], h=w["h"], n=w["n"], v=w["v"], num_layers=w["layers"])
            model = sg.MeshModel(mesh, cfg, None, seed=1234)
            ws = model.make_workspace()
            rng = np.random.default_rng(1)
            tok = torch.from_numpy(rng.integers(0, cfg.v, (b, cfg.s))).cuda()
            lab = torch.from_numpy(rng.integers(0, cfg.v, (b, cfg.s))).cuda()
            if args.mode == "infer":
                model.infer(tok, lab, ws)
            else:
                model.train_step(tok, lab, ws, 1e-4, checkpointing=args.checkpointing)
            torch.cuda.synchronize()
        except torch.cuda.OutOfMemoryError:
            ok = False
        del model, ws, tok, lab
        gc.collect()
        torch.cuda.empty_cache()
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([1.0 if ok else 0.0], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MIN)
            ok = bool(t.item() > 0.5)
        return ok

    tried = {}
    lo, hi = 0, None
    b = max(w["b"], r)
    while hi is None and b <= 1 << 16:
        tried[b] = fits(b)
        if tried[b]:
            lo, b = b, 2 * b
        else:
            hi = b
    while hi is not None and hi - lo > max(r, lo // 8):
        mid = (lo + hi) // 2 // r * r
        if mid <= lo:
            break
        tried[mid] = fits(mid)
        lo, hi = (mid, hi) if tried[mid] else (lo, mid)
    return {"max_batch": lo, "first_oom": hi, "probes": {str(k): v for k, v in sorted(tried.items())},
            "mode": args.mode, "hbm_gb": torch.cuda.get_device_properties(0).total_memory / 1e9}


def summa_point(sg, K, mesh, n, pk, barrier, world) -> dict:
    """TFLOP/s of the three SUMMA forms at N x N x N bf16 on the bench mesh."""
    import torch

    out = {"N": n, "mesh": f"{mesh.r}x{mesh.c}", "peak": pk["bf16_burst"], "peak_source": pk["src"] + " burst bf16"}
    ws = sg.Workspace(mesh.p)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(0)

    def rand_mat(layout):
        m = sg.ShardedMatrix(mesh, n, n, [None] * (mesh.r * mesh.c if layout == "act" else mesh.c * mesh.c), layout)
        gr, gc = m.grid
        for k in range(gr * gc):
            if mesh.owns(m.owner(k // gc, k % gc)):
                m.blocks[k] = torch.randn(n // gr, n // gc, device="cuda", generator=gen).bfloat16()
        return m

    A, W, A2 = rand_mat("act"), rand_mat("weight"), rand_mat("act")
    forms = {"ab": lambda: sg.summa_ab(A, W, ws, out_dtype=torch.bfloat16),
             "abt": lambda: sg.summa_abt(A, W, ws, out_dtype=torch.bfloat16),
             "atb": lambda: sg.summa_atb(A, A2, ws)}
    flops_dev = 2.0 * n ** 3 / mesh.p
    for name, fn in forms.items():
        for _ in range(2):
            fn()
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        iters = 10
        e0.record()
        for _ in range(iters):
            fn()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / iters
        if world > 1:
            import torch.distributed as dist

            t = torch.tensor([ms], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        tf = 2.0 * n ** 3 / (ms * 1e-3) / 1e12
        out[name] = {"ms": ms, "tflops": tf, "tflops_per_gpu": flops_dev / (ms * 1e-3) / 1e12,
                     "frac": flops_dev / (ms * 1e-3) / 1e12 / pk["bf16_burst"]}
    return out


if __name__ == "__main__":
    main()
