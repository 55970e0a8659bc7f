"""Group an ncu SASS source dump (--page source --csv --print-source sass)
into runs of equal execution count: where the warp instructions go.
usage: ncu_segments.py src.csv [min_pct]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
mn = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
hdr, data = rows[1], rows[2:]
isrc = hdr.index("Source")
iex = hdr.index("Instructions Executed")
iss = hdr.index("Warp Stall Sampling (All Samples)")
tot = sum(int(r[iex]) for r in data if r[iex].isdigit())
tots = sum(int(r[iss]) for r in data if r[iss].isdigit())
print("total warp instructions", tot, "samples", tots)
segs, cur = [], None
for k, r in enumerate(data):
    ex = int(r[iex]) if r[iex].isdigit() else 0
    if cur is None or ex != cur[0]:
        if cur:
            segs.append(cur)
        cur = [ex, k, k, 0]
    cur[2] = k
    cur[3] += int(r[iss]) if r[iss].isdigit() else 0
segs.append(cur)
for ex, a, b, smp in segs:
    n = b - a + 1
    if ex * n > tot * mn / 100 or smp > tots * mn / 100:
        print(f"lines {a:5d}-{b:5d} n={n:4d} exec/line={ex:8d} "
              f"instr={ex * n / tot * 100:5.1f}% samples={smp / tots * 100:5.1f}% "
              f"first={data[a][isrc].strip()[:40]}")
