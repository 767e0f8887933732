"""Opcode histogram (executed warp instructions) from `ncu --page source --csv --print-source cuda,sass`.
usage: ncu_opcode_hist.py source.csv [divisor]   (divisor: e.g. matrices*steps*warps for per-warp-step counts)"""
import collections
import csv
import re
import sys

ops = collections.Counter()
stalls = collections.Counter()
tot = 0.0
for r in csv.reader(open(sys.argv[1])):
    if len(r) < 8 or r[0] != "" or not r[2].startswith("0x"):
        continue
    try:
        n = float(r[7])
        st = float(r[4])
    except ValueError:
        continue
    src = r[3].strip()
    m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_]+)", src)
    op = m.group(2) if m else src[:10]
    ops[op] += n
    stalls[op] += st
    tot += n
div = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
print(f"warp instructions {tot:.0f}")
for k, v in ops.most_common(32):
    print(f"{k:12s} {v/1e6:9.2f}M {100*v/tot:5.1f}%   {v/div:8.1f}   stall samples {stalls[k]:.0f}")
