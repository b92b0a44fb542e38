"""Per-kernel HBM evidence for the non-GEMM kernels of one training step.

    python tools/summarize_rowops.py rowops.csv tag [hbm_gbs]

Input: ncu --csv of --metrics gpu__time_duration.sum,dram__bytes_read.sum,
dram__bytes_write.sum over tools/one_step.py, filtered to the row kernels. Output:
profiles/<tag>_rowops_ncu.csv with launches, mean duration, mean DRAM bytes and the
achieved DRAM GB/s (and fraction of the measured copy bandwidth) per kernel.
"""
import collections
import json
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent))
from summarize_ncu import rows, to_unit  # noqa: E402


def main():
    path, tag = sys.argv[1], sys.argv[2]
    peak = float(sys.argv[3]) if len(sys.argv) > 3 else json.loads(
        (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6459.3)
    per = collections.defaultdict(dict)
    for r in rows(path):
        per[r["ID"]]["kernel"] = r["Kernel Name"].split("(")[0]
        per[r["ID"]][r["Metric Name"]] = to_unit(r["Metric Value"], r["Metric Unit"], "")
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for v in per.values():
        a = agg[v["kernel"]]
        a[0] += 1
        a[1] += v.get("gpu__time_duration.sum", 0.0)
        a[2] += v.get("dram__bytes_read.sum", 0.0) + v.get("dram__bytes_write.sum", 0.0)
    out = [f"# {tag}: ncu per-launch DRAM bytes and duration of the non-GEMM kernels of one BERT-large 1x1 step",
           f"# (cold cache, serialised; achieved = dram bytes / duration vs {peak:.0f} GB/s measured copy bandwidth)",
           "kernel,launches,mean_us,mean_dram_MB,achieved_GBs,frac_of_hbm"]
    for k, (n, us, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        gbs = by / (us * 1e-6) / 1e9 if us > 0 else 0.0
        out.append(f"{k},{n},{us / n:.2f},{by / n / 1e6:.2f},{gbs:.0f},{gbs / peak:.3f}")
    Path(f"profiles/{tag}_rowops_ncu.csv").write_text("\n".join(out) + "\n")
    print("\n".join(out))


if __name__ == "__main__":
    main()
