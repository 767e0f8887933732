"""Per source line, which opcodes were executed: top lines for the given opcodes.
usage: ncu_line_ops.py source.csv OP [OP...]"""
import collections
import csv
import re
import sys

cur = None
f = "?"
per = collections.defaultdict(collections.Counter)
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        f = r[1].split("/")[-1]
        continue
    if len(r) < 8:
        continue
    if r[0] not in ("", "Line No", "Function Name"):
        try:
            cur = (f, int(r[0]), r[1].strip()[:70])
        except ValueError:
            pass
        continue
    if r[0] == "" and r[2].startswith("0x") and cur:
        try:
            n = float(r[7])
        except ValueError:
            continue
        m = re.match(r"(@!?U?P\d+\s+)?([A-Z0-9_]+)", r[3].strip())
        per[cur][m.group(2) if m else "?"] += n
for op in sys.argv[2:]:
    print("==", op)
    rows = sorted(((c[op], k) for k, c in per.items() if c[op] > 0), reverse=True)[:12]
    for n, k in rows:
        print(f"  {n/1e6:7.2f}M  {k[0]}:{k[1]}  {k[2]}")
