"""Summarise an ncu --page source --print-source sass CSV: hottest SASS lines by stall samples."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
data = rows[2:]
def num(r, k):
    try:
        return float(r[ix[k]])
    except (ValueError, KeyError, IndexError):
        return 0.0
tot_s = sum(num(r, "Warp Stall Sampling (All Samples)") for r in data)
tot_i = sum(num(r, "Instructions Executed") for r in data)
print(f"lines {len(data)} stall samples {tot_s:.0f} warp-instructions {tot_i:.0f}")
top = sorted(data, key=lambda r: -num(r, "Warp Stall Sampling (All Samples)"))[: int(sys.argv[2]) if len(sys.argv) > 2 else 40]
for r in top:
    print(f"{num(r,'Warp Stall Sampling (All Samples)'):8.0f} {num(r,'Instructions Executed'):10.0f}  {r[ix['Address']][-5:]}  {r[ix['Source']].strip()[:90]}")
