"""Print the per-role timeline captured by SFHR_TC_TRACE=1 (tools/tc_trace.py output)."""
import sys

lines = [l for l in open(sys.argv[1]) if l.startswith('[tc-trace]')]
blocks = []
for l in lines:
    if 'B=' in l:
        blocks.append({'hdr': l.strip()})
        continue
    role = int(l.split('role')[1].split(':')[0])
    blocks[-1][role] = [int(v) for v in l.split(':', 1)[1].split()]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 12
for b in blocks:
    print(b['hdr'])
    for role, name in ((0, 'producers'), (1, 'MMA'), (2, 'E_A'), (3, 'E_B')):
        v = b.get(role, [])
        print(f"  {name:9s}", ' '.join(f"{x:6d}" for x in v[:n]))
    P = b.get(0, [])
    EB = b.get(3, [])
    if EB:
        print(f"  E_B end of trace {EB[-1]} cycles over {len(EB) // 3} steps -> {EB[-1] / max(1, len(EB) // 3):.0f} / step")
