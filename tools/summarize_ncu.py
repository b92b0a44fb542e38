"""Summaries of the ncu CSVs into profiles/: per-kernel launch shares and the
GEMM's per-launch DRAM traffic (python tools/summarize_ncu.py launches.csv gemm_traffic.csv tag)."""
import collections
import csv
import json
import sys
from pathlib import Path


def rows(path):
    lines = Path(path).read_text().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    return list(csv.DictReader(lines[start:]))


def to_unit(v, unit, want):
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "msecond": 1e3, "byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6,
             "Gbyte": 1e9}
    return float(v.replace(",", "")) * scale.get(unit, 1.0)


def main():
    launches, traffic, tag = sys.argv[1], sys.argv[2], sys.argv[3]
    agg = collections.defaultdict(lambda: [0, 0.0])
    for r in rows(launches):
        if r["Metric Name"] != "gpu__time_duration.sum":
            continue
        name = r["Kernel Name"]
        base = name.split("(")[0]
        agg[base][0] += 1
        agg[base][1] += to_unit(r["Metric Value"], r["Metric Unit"], "us")
    total = sum(v[1] for v in agg.values())
    out = [f"# ncu launch list of one BERT-large 1x1 training step (tools/one_step.py), {tag}",
           "# ncu --metrics gpu__time_duration.sum --clock-control none: serialised, cold-cache per launch;",
           f"# total {total / 1e3:.2f} ms over {sum(v[0] for v in agg.values())} launches; compare SHARES with bench.py",
           "kernel,launches,total_us,share"]
    for name, (n, us) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        out.append(f"{name},{n},{us:.1f},{100 * us / total:.1f}%")
    gemm_us = sum(us for name, (n, us) in agg.items() if "gemm_kernel" in name)
    out.append(f"# sg_gemm (all tcgen05 GEMM instantiations) share: {100 * gemm_us / total:.1f}%")
    Path(f"profiles/{tag}_launches_summary.csv").write_text("\n".join(out) + "\n")
    per = collections.defaultdict(dict)
    for r in rows(traffic):
        per[r["ID"]]["kernel"] = r["Kernel Name"].split("(")[0]
        per[r["ID"]][r["Metric Name"]] = to_unit(r["Metric Value"], r["Metric Unit"], "")
    n = len(per)
    rd = sum(v.get("dram__bytes_read.sum", 0.0) for v in per.values())
    wr = sum(v.get("dram__bytes_write.sum", 0.0) for v in per.values())
    t = sum(v.get("gpu__time_duration.sum", 0.0) for v in per.values())
    tens = [v.get("sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", 0.0) for v in per.values()]
    summary = {"tag": tag, "kernel": "sg::gemm_kernel (all instantiations, one training step)", "launches": n,
               "dram_read_bytes": rd, "dram_write_bytes": wr, "traffic_bytes_per_launch": (rd + wr) / max(n, 1),
               "gpu_time_us": t, "tensor_pipe_active_pct_time_weighted":
                   sum(x * v.get("gpu__time_duration.sum", 0.0) for x, v in zip(tens, per.values())) / max(t, 1e-9),
               "source": "ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,"
                         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed -k regex:gemm_kernel"}
    Path(f"profiles/{tag}_gemm_traffic.json").write_text(json.dumps(summary, indent=1) + "\n")
    print("\n".join(out[:25]))
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
