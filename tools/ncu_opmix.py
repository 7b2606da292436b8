"""Instruction mix (per SASS opcode) of an ncu report's first kernel: python tools/ncu_opmix.py rep.ncu-rep"""
import collections
import csv
import io
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
ie, src, smp = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ops, samples, tot = collections.Counter(), collections.Counter(), 0
for r in rows[2:]:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    toks = r[src].split()
    if not toks:
        continue
    op = (toks[1] if toks[0].startswith("@") else toks[0]).split(".")[0]
    ops[op] += int(r[ie])
    samples[op] += int(r[smp] or 0)
    tot += int(r[ie])
print("warp instructions", tot)
for op, n in ops.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {100 * n / tot:5.1f}%  stall samples {samples[op]}")
