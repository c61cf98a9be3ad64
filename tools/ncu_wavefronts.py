"""Shared-memory and global wavefronts per SASS opcode class for one kernel of an ncu report
(from the source page's per-instruction counters).  usage: ncu_wavefronts.py REP [KERNEL_SUBSTR]"""
import collections
import csv
import io
import re
import subprocess
import sys

rep, want = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "")
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
for b in out.split('"Kernel Name",')[1:]:
    name = b.split("\n", 1)[0]
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    if "L1 Wavefronts Shared" not in h:
        continue
    col = {k: h.index(k) for k in ("Source", "Instructions Executed", "L1 Wavefronts Shared",
                                   "L1 Wavefronts Shared Ideal", "L2 Theoretical Sectors Global", "L1 Tag Requests Global")}
    agg = collections.defaultdict(lambda: [0, 0, 0, 0, 0])
    for r in rows[1:]:
        if len(r) <= max(col.values()):
            continue
        src = r[col["Source"]].strip()
        op = re.sub(r"^@!?U?P\w+\s+", "", src).split(" ")[0]
        a = agg[op]
        a[0] += int(r[col["Instructions Executed"]] or 0)
        a[1] += int(r[col["L1 Wavefronts Shared"]] or 0)
        a[2] += int(r[col["L1 Wavefronts Shared Ideal"]] or 0)
        a[3] += int(r[col["L2 Theoretical Sectors Global"]] or 0)
        a[4] += int(r[col["L1 Tag Requests Global"]] or 0)
    print(f"== {name[:90]}")
    print(f"{'op':28s} {'inst':>12s} {'smem_wf':>12s} {'smem_ideal':>12s} {'l2_sect':>12s} {'l1_tagreq':>12s}")
    for op, a in sorted(agg.items(), key=lambda kv: -(kv[1][1] + kv[1][3])):
        if a[1] + a[3] + a[4] == 0:
            continue
        print(f"{op:28s} {a[0]:12d} {a[1]:12d} {a[2]:12d} {a[3]:12d} {a[4]:12d}")
