"""Opcode histogram of a SASS dump (cuobjdump -sass), optionally restricted to an address range."""
import re
import sys
from collections import Counter

txt = open(sys.argv[1]).read().splitlines()
lo = int(sys.argv[2], 16) if len(sys.argv) > 2 else 0
hi = int(sys.argv[3], 16) if len(sys.argv) > 3 else 1 << 60
c = Counter()
pat = re.compile(r"/\*([0-9a-f]{4,})\*/\s+(@!?U?P[T0-9]+\s+)?([A-Z][A-Z0-9_]*)(\.[A-Z0-9_.]+)?")
for ln in txt:
    m = pat.search(ln)
    if not m:
        continue
    a = int(m.group(1), 16)
    if lo <= a < hi:
        c[m.group(3)] += 1
tot = sum(c.values())
print("total", tot)
for k, v in c.most_common(45):
    print(f"{k:10s} {v}")
