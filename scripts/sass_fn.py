"""Extract one kernel's SASS from `cuobjdump -sass` output and histogram opcodes.

    cuobjdump -sass lib.so > all.sass; python scripts/sass_fn.py all.sass <substring>
"""
import re
import sys
from collections import Counter

path, pat = sys.argv[1], sys.argv[2]
text = open(path).read().split("\n")
out, on = [], False
for line in text:
    if "Function :" in line:
        on = pat in line
        if on:
            out.append(line)
        continue
    if on:
        out.append(line)
ops = Counter()
for line in out:
    m = re.match(r"\s+/\*[0-9a-f]+\*/\s+(@!?U?P\w+\s+)?([A-Z0-9_]+)", line)
    if m:
        ops[m.group(2)] += 1
print(out[0] if out else "not found")
print(sum(ops.values()), "instructions")
for op, n in ops.most_common(30):
    print(f"{n:6d} {op}")
if len(sys.argv) > 3:
    print("\n".join(out))
