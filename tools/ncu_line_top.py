"""Per CUDA source line totals from `ncu --page source --csv --print-source cuda,sass`."""
import csv
import sys

fname = None
agg = {}
for row in csv.reader(open(sys.argv[1])):
    if not row:
        continue
    if row[0] == "File Path":
        fname = row[1].split("/")[-1]
        continue
    if row[0] in ("Function Name", "Line No"):
        if row[0] == "Line No":
            hdr = row
            ix = {h: i for i, h in enumerate(hdr)}
        continue
    try:
        line = int(row[0])
    except ValueError:
        continue
    def num(k):
        try:
            return float(row[ix[k]])
        except (ValueError, KeyError):
            return 0.0
    key = (fname, line)
    a = agg.setdefault(key, [0.0, 0.0, row[1].strip()[:80]])
    a[0] += num("Warp Stall Sampling (All Samples)")
    a[1] += num("Instructions Executed")
tot = [sum(v[0] for v in agg.values()), sum(v[1] for v in agg.values())]
print(f"stall samples {tot[0]:.0f}  warp instructions {tot[1]:.0f}")
key = 1 if len(sys.argv) > 3 and sys.argv[3] == "inst" else 0
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][key])[: int(sys.argv[2]) if len(sys.argv) > 2 else 30]:
    print(f"{v[0]:7.0f} {100*v[0]/max(tot[0],1):5.1f}%  {v[1]:11.0f} {100*v[1]/max(tot[1],1):5.1f}%  {k[0]}:{k[1]}  {v[2]}")
