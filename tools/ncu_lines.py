"""Per-source-line warp-stall summary of an ncu report (ncu --page source --print-source cuda,sass).

    python tools/ncu_lines.py REPORT.ncu-rep [top]
"""
import csv
import io
import subprocess
import sys


def main():
    rep, top = sys.argv[1], int(sys.argv[2]) if len(sys.argv) > 2 else 30
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    agg, fname = {}, ""
    h = None
    for r in rows:
        if r and r[0] == "File Path":
            fname = r[1].split("/")[-1]
        elif r and r[0] == "Line No":
            h = {n: i for i, n in enumerate(r)}
            stalls = [n for n in r if n.startswith("stall_") and "Not Issued" not in n]
        elif h and r and r[0].isdigit() and r[2] == "-":  # source line rows (not per-SASS rows)
            key = (fname, int(r[0]))
            s = float(r[h["Warp Stall Sampling (All Samples)"]] or 0)
            det = {n[6:]: float(r[h[n]] or 0) for n in stalls}
            agg[key] = (s, r[1].strip(), det, float(r[h["Instructions Executed"]] or 0))
    tot = sum(v[0] for v in agg.values())
    print(f"total samples {tot:.0f}")
    for (f, ln), (s, src, det, ie) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
        d = sorted(det.items(), key=lambda kv: -kv[1])[:3]
        print(f"{f}:{ln:<5} {s / tot * 100:5.1f}% inst {ie:10.0f}  {src[:60]:60s} "
              + " ".join(f"{k}={v / max(s, 1) * 100:.0f}%" for k, v in d))


if __name__ == "__main__":
    main()
