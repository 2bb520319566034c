"""Instruction histogram of the innermost loop containing a given SASS opcode.

python tools/sass_loop.py <file.sass> [OPCODE]   (cuobjdump -sass -fun <kernel> output)
Picks the backward-branch range holding the most OPCODE instructions (the column
loop) and prints its opcode counts.
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
keys = [a for a, op, _ in ins if op.startswith(key)]
rngs = []  # backward-branch ranges
for a, op, rest in ins:
    if op.startswith("BRA"):
        t = re.search(r"0x([0-9a-f]+)", rest)
        if t and int(t.group(1), 16) < a:
            tgt = int(t.group(1), 16)
            rngs.append((tgt, a, sum(tgt <= k <= a for k in keys)))
top = max(n for _, _, n in rngs)
# the smallest loop holding >= 90 % of the most OPCODE instructions any loop holds
lo, hi, _ = min((r for r in rngs if r[2] >= 0.9 * top), key=lambda r: r[1] - r[0])
c = Counter(op for a, op, _ in ins if lo <= a <= hi)
print(f"loop 0x{lo:x}..0x{hi:x}: {sum(c.values())} instructions")
for op, n in c.most_common():
    print(f"{n:6d} {op}")
