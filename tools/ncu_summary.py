"""Summarise an ncu report: key metrics + SASS opcode mix per kernel (for profiles/)."""
import collections, csv, io, re, subprocess, sys

rep = sys.argv[1]
KEYS = ["Duration", "DRAM Throughput", "Memory Throughput", "L1/TEX Hit Rate", "L2 Hit Rate",
        "Compute (SM) Throughput", "Achieved Occupancy", "Theoretical Occupancy", "Registers Per Thread",
        "Block Size", "Grid Size", "Dynamic Shared Memory Per Block", "L1/TEX Cache Throughput",
        "L2 Cache Throughput", "Issue Slots Busy", "Executed Ipc Active", "Warp Cycles Per Issued Instruction"]
RAW = re.compile(r"^(dram__bytes_(read|write)\.sum|smsp__inst_executed\.sum|lts__t_sectors_srcunit_tex_op_read\.sum|"
                 r"l1tex__data_pipe_lsu_wavefronts_mem_shared\.sum|l1tex__t_sectors_pipe_lsu_mem_global_op_ld\.sum|"
                 r"l1tex__data_bank_conflicts_pipe_lsu_mem_shared\.sum|lts__t_sector_hit_rate\.pct|"
                 r"smsp__pcsamp_warps_issue_stalled_(long_scoreboard|short_scoreboard|wait|barrier|branch_resolving|"
                 r"mio_throttle|lg_throttle|math_pipe_throttle|not_selected|selected|no_instruction|membar|sleeping))$")


def run(*a):
    return subprocess.run(["ncu", "-i", rep, *a], capture_output=True, text=True).stdout


det = list(csv.reader(io.StringIO(run("--page", "details", "--csv"))))
h = det[0]
ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
per = collections.OrderedDict()
for r in det[1:]:
    if r[mi] in KEYS:
        per.setdefault(r[ki], {})[r[mi]] = f"{r[vi]} {r[ui]}".strip()
raw = list(csv.reader(io.StringIO(run("--page", "raw", "--csv"))))
rh = raw[0]
names = [row[rh.index("Kernel Name")] for row in raw[2:]]
rawv = collections.OrderedDict()
for j, col in enumerate(rh):
    if RAW.match(col):
        for n, row in zip(names, raw[2:]):
            rawv.setdefault(n, {})[col] = f"{row[j]} {raw[1][j]}".strip()
for k, m in per.items():
    print(f"== {k}")
    for key in KEYS:
        if key in m:
            print(f"   {key:40s} {m[key]}")
    for key, v in rawv.get(k, {}).items():
        print(f"   {key:60s} {v}")
src = list(csv.reader(io.StringIO(run("--page", "source", "--csv", "--print-source", "sass"))))
cur = None
mix = collections.OrderedDict()
hdr = None
for r in src:
    if r and r[0] == "Kernel Name":
        cur = r[1]
        mix[cur] = (collections.Counter(), collections.Counter())
        continue
    if r and r[0] == "Address":
        hdr = r
        continue
    if cur and hdr and len(r) == len(hdr) and r[hdr.index("Instructions Executed")].isdigit():
        m = re.match(r"\s*(@!?U?P\w+\s+)?([A-Z0-9_]+)", r[hdr.index("Source")])
        op = m.group(2) if m else "?"
        mix[cur][0][op] += int(r[hdr.index("Instructions Executed")])
        mix[cur][1][op] += int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
for k, (ins, st) in mix.items():
    tot, sa = sum(ins.values()), max(1, sum(st.values()))
    print(f"== SASS mix {k[:70]}  total warp-inst {tot}")
    print("   " + "  ".join(f"{o} {c / tot * 100:.1f}%/{st[o] / sa * 100:.0f}%s" for o, c in ins.most_common(16)))
