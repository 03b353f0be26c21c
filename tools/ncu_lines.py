"""Per-CUDA-source-line digest of an ncu report: instructions executed and warp-stall samples
per line (compile with -lineinfo, capture with --import-source on).

    python tools/ncu_lines.py REPORT.ncu-rep [N]
"""
import csv
import subprocess
import sys

path = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", path, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, recs = "?", None, []
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname, hdr = r[1].split("/")[-1], None
        continue
    if r[0] == "Line No":
        hdr = r
        iS, iE = hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
        continue
    if hdr is None or r[2] != "-":   # cuda rows carry "-" in the Address column
        continue
    try:
        recs.append((float(r[iE] or 0), float(r[iS] or 0), fname, r[0], r[1].strip()[:90]))
    except (ValueError, IndexError):
        pass
tot_e = sum(x[0] for x in recs)
tot_s = sum(x[1] for x in recs)
print(f"total inst executed {tot_e:.4g}, samples {tot_s:.4g}")
for e, s, f, ln, src in sorted(recs, reverse=True)[:n]:
    print(f"{100 * e / tot_e:6.2f}% ex {100 * s / max(tot_s, 1):6.2f}% smp  {f}:{ln:5s} {src}")
