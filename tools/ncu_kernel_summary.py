"""One-line summaries of ncu --set full reports (duration, tensor pipe, smem wavefronts,
MUFU, issue slots, DRAM, top stall reasons): python tools/ncu_kernel_summary.py rep.ncu-rep ..."""
import csv
import io
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_pipe_active_pct",
    "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "tc_smem_wavefronts_pct",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed": "lsu_smem_wavefronts_pct",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_elapsed": "xu(MUFU)_inst_pct",
    "sm__instruction_throughput.avg.pct_of_peak_sustained_active": "issue_slots_busy_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
}


def summarize(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    head, units, vals = rows[0], rows[1], rows[2]
    d = dict(zip(head, vals))
    u = dict(zip(head, units))
    res = {"kernel": d.get("Kernel Name", "?").split("(")[0]}
    for k, name in KEYS.items():
        v = d.get(k, "")
        try:
            x = float(v.replace(",", ""))
            if k == "gpu__time_duration.sum":
                x = x / 1000.0 if u.get(k) in ("nsecond", "ns") else (x * 1000.0 if u.get(k) in ("msecond", "ms") else x)
            res[name] = f"{x:.2f}"
        except ValueError:
            res[name] = "n/a"
    stalls = {k.split("issue_stalled_")[1].split("_per_")[0]: float(v.replace(",", "") or 0)
              for k, v in d.items() if k.startswith("smsp__average_warps_issue_stalled_") and
              k.endswith("_per_issue_active.ratio") and "not_issued" not in k}
    tot = sum(stalls.values()) or 1.0
    top = sorted(stalls.items(), key=lambda kv: -kv[1])[:4]
    res["top_stalls"] = " ".join(f"{k}:{v / tot * 100:.0f}%" for k, v in top)
    return res


if __name__ == "__main__":
    rs = [summarize(r) for r in sys.argv[1:]]
    cols = ["kernel", *KEYS.values(), "top_stalls"]
    print(",".join(cols))
    for r in rs:
        print(",".join(r[c] for c in cols))
