"""Per-chunk pipeline timeline from BM_TIMELINE=2 stderr lines ([tl] kind start end)."""
import sys
import numpy as np
rows = [l.split()[1:] for l in open(sys.argv[1]) if l.startswith("[tl]")]
# the last run's records: restart when a Lloyd graph starts at 0
start = max(i for i, r in enumerate(rows) if r[0] == "1" and float(r[1]) == 0.0)
rows = [(int(k), float(a), float(b)) for k, a, b in rows[start - 1 if start else 0:]]
lloyd = [r for r in rows if r[0] == 1]
prep = [r for r in rows if r[0] == 0]
spec = [r for r in rows if r[0] == 2]
c0 = int(sys.argv[2]) if len(sys.argv) > 2 else 40
print("chunk  lloyd[start,end]   prep(c+1)[start,end]   spec(c+1)[start,end]   (us)")
for c in range(c0, c0 + 12):
    L = lloyd[c]
    P = prep[c + 1] if c + 1 < len(prep) else (0, 0, 0)
    S = spec[c] if c < len(spec) else (0, 0, 0)
    print(f"{c:4d}  {L[1]:9.1f} {L[2]:9.1f}   {P[1]:9.1f} {P[2]:9.1f}   {S[1]:9.1f} {S[2]:9.1f}")
