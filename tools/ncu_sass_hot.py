"""Hot SASS of one kernel in an ncu report: instructions executed and stall samples per
instruction, in program order around the hottest region.  usage: ncu_sass_hot.py REP [KERNEL_SUBSTR] [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
want = sys.argv[2] if len(sys.argv) > 2 else ""
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True, text=True).stdout
blocks = out.split('"Kernel Name",')
for b in blocks[1:]:
    name = b.split("\n", 1)[0]
    if want not in name:
        continue
    rows = list(csv.reader(io.StringIO(b.split("\n", 1)[1])))
    h = rows[0]
    ia, isrc, iex, ismp = h.index("Address"), h.index("Source"), h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
    ith = h.index("Avg. Predicated-On Threads Executed")
    data = [(r[ia], r[isrc].strip(), int(r[iex] or 0), int(r[ismp] or 0), r[ith]) for r in rows[1:] if len(r) > ismp]
    tot = sum(d[2] for d in data)
    tots = sum(d[3] for d in data)
    print(f"== {name[:100]}  inst {tot}  samples {tots}")
    hot = sorted(range(len(data)), key=lambda i: -data[i][2])[:top]
    for i in sorted(hot):
        a, s, e, sm, th = data[i]
        print(f"{i:5d} {e / tot * 100:5.1f}% {sm / max(tots, 1) * 100:5.1f}%s thr{th:>5s}  {s}")
