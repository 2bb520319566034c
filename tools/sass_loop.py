"""Instruction histogram of the innermost loop containing a given SASS opcode.

python tools/sass_loop.py <file.sass> [OPCODE]   (cuobjdump -sass -fun <kernel> output)
Finds every backward branch whose range covers the first OPCODE instruction and
prints the opcode counts of the smallest such range (the column loop).
"""
import re
import sys
from collections import Counter

path = sys.argv[1]
key = sys.argv[2] if len(sys.argv) > 2 else "VIMNMX3"
ins = []
for line in open(path):
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_.]+)(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(3), m.group(4)))
hot = next(a for a, op, _ in ins if op.startswith(key))
best = None
for a, op, rest in ins:
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if t:
            tgt = int(t.group(1), 16)
            if tgt <= hot <= a and (best is None or a - tgt < best[1] - best[0]):
                best = (tgt, a)
lo, hi = best
c = Counter(op for a, op, _ in ins if lo <= a <= hi)
print(f"loop 0x{lo:x}..0x{hi:x}: {sum(c.values())} instructions")
for op, n in c.most_common():
    print(f"{n:6d} {op}")
