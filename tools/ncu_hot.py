"""Summarise an ncu --page source --csv export: hottest SASS lines by warp
stall samples (usage: ncu -i rep --page source --csv -k regex:K > f.csv;
python tools/ncu_hot.py f.csv [top])."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
hdr = rows[1]
ci = {h: i for i, h in enumerate(hdr)}
data = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    w = float(r[ci["Warp Stall Sampling (All Samples)"]] or 0)
    data.append((w, r[ci["Address"]][-5:], r[ci["Source"]].strip()[:70],
                 r[ci["Instructions Executed"]]))
tot = sum(x[0] for x in data) or 1
print("total samples", tot)
for w, a, s, e in sorted(data, key=lambda x: -x[0])[:top]:
    print(f"{w / tot:6.3f} {a} {e:>10} {s}")
