"""Summarise an `ncu --page source --csv` dump: hottest SASS instructions and stall totals.

    ncu -i rep.ncu-rep --page source --csv --launch-skip S --launch-count 1 > src.csv
    python tools/ncu_hot.py src.csv [top]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hdr = rows[1]
ix = {h: i for i, h in enumerate(hdr)}
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = Counter()
lines = []
for r in rows[2:]:
    if len(r) < len(hdr):
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    except ValueError:
        continue
    st = {h: int(r[ix[h]] or 0) for h in stall_cols}
    tot.update(st)
    lines.append((s, r[ix["Address"]], r[ix["Source"]], st, r[ix["Instructions Executed"]]))
S = sum(l[0] for l in lines) or 1
print("total samples", S)
print("stalls:", ", ".join(f"{k[6:]}={v / S:.1%}" for k, v in tot.most_common(10)))
for s, a, src, st, ex in sorted(lines, key=lambda x: -x[0])[:top]:
    big = ", ".join(f"{k[6:]}={v}" for k, v in Counter(st).most_common(3) if v)
    print(f"{s / S:6.2%} {a:>6} {src[:60]:60s} ex={ex:>10} {big}")
