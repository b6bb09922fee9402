"""Per-CUDA-source-line stall samples from `ncu --page source --csv --print-source cuda,sass`.

    python tools/ncu_lines.py src.csv [top]
"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if r and r[0] == "Line No")
hdr = rows[hi]
ix = {}
for i, h in enumerate(hdr):
    ix.setdefault(h, i)
stall = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
lines = []
for r in rows[hi + 1:]:
    if len(r) < len(hdr) or not r[0]:
        continue
    try:
        s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
        ex = int(r[ix["Instructions Executed"]] or 0)
    except ValueError:
        continue
    st = Counter({h[6:]: int(r[ix[h]] or 0) for h in stall})
    lines.append((s, int(r[0]), r[1].strip(), ex, st))
S = sum(l[0] for l in lines) or 1
E = sum(l[3] for l in lines) or 1
print(f"samples {S}  warp-instructions {E}")
for s, ln, src, ex, st in sorted(lines, key=lambda x: -x[0])[:top]:
    big = ", ".join(f"{k}={v / max(s, 1):.0%}" for k, v in st.most_common(3) if v)
    print(f"{s / S:6.2%} ex {ex / E:6.2%} L{ln:<4d} {src[:70]:70s} {big}")
