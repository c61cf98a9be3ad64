"""Per-CUDA-source-line instruction and stall-sample totals of one kernel in an ncu report
(lines that carry metrics in the cuda,sass source view).  usage: ncu_lines.py REP [KERNEL_SUBSTR] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows, fname, func = [], "", ""
for line in out.splitlines():
    if line.startswith('"File Path"'):
        fname = line.split('","')[1].rstrip('"').rsplit("/", 1)[-1]
        continue
    if line.startswith('"Function Name"'):
        func = line.split('","')[1].rstrip('"')
        continue
    if line.startswith('"Line No"'):
        hdr = next(csv.reader([line]))
        continue
    r = next(csv.reader([line]))
    if len(r) < 8 or r[2] != "-" or want not in func:
        continue
    rows.append((fname, r[0], r[1], float(r[hdr.index("Instructions Executed")] or 0),
                 float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)))
ti = sum(r[3] for r in rows) or 1
ts = sum(r[4] for r in rows) or 1
print(f"instructions {ti:.4g}  samples {ts:.4g}")
for f, ln, src, ins, smp in sorted(rows, key=lambda r: -r[3])[:top]:
    print(f"{ins / ti * 100:5.1f}% inst {smp / ts * 100:5.1f}% smp  {f}:{ln:<5} {src.strip()[:100]}")
