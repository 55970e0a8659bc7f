"""Summarise an ncu --page source --csv --print-source sass dump: hottest
SASS lines with their dominant stall reasons.  usage: ncu_hot.py src.csv [N]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
iss = hdr.index("Warp Stall Sampling (All Samples)")
iex = hdr.index("Instructions Executed")
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = sum(int(r[iss]) for r in data if r[iss].isdigit())
agg = {}
for r in data:
    for h in reasons:
        v = r[hdr.index(h)]
        if v.isdigit():
            agg[h] = agg.get(h, 0) + int(v)
print("total samples", tot, "executed warp-instr",
      sum(int(r[iex]) for r in data if r[iex].isdigit()))
print("by reason:", sorted(((v, k) for k, v in agg.items()), reverse=True)[:8])
rank = sorted(range(len(data)), key=lambda k: -int(data[k][iss])
              if data[k][iss].isdigit() else 0)[:n]
for k in sorted(rank):
    r = data[k]
    why = sorted(((int(r[hdr.index(h)]), h[6:]) for h in reasons
                  if r[hdr.index(h)].isdigit() and int(r[hdr.index(h)]) > 0),
                 reverse=True)[:2]
    print(f"{k:5d} {r[iss]:>6} {r[iex]:>9} {r[isrc].strip()[:60]:60s} {why}")
