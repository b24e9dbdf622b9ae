"""Dynamic SASS opcode mix of one kernel from an ncu report (SourceCounters section):
    python tools/ncu_opmix.py report.ncu-rep [warps]   (warps: divide counts per warp)"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, st = h.index("Instructions Executed"), h.index("Warp Stall Sampling (All Samples)")
warps = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
by, ss, tot = collections.Counter(), collections.Counter(), 0
for x in rows[2:]:
    if len(x) <= max(ie, st) or not x[ie].strip().isdigit():
        continue  # another kernel's header / section line
    toks = x[1].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0])
    n = int(x[ie] or 0)
    by[op] += n
    ss[op] += int(x[st] or 0)
    tot += n
print(f"total {tot}  per-warp {tot / warps:.1f}")
for op, n in by.most_common(30):
    print(f"{op:24s} {n / warps:8.1f}  stall_samples {ss[op]}")
