"""Instruction mix of the loops (backward branches) of one kernel's SASS.
    cuobjdump -sass lib.so > /tmp/all.sass; python tools/sass_loops.py /tmp/all.sass <name-substring> [min_bytes]"""
import re
import sys
from collections import Counter

path, pat = sys.argv[1], sys.argv[2]
minb = int(sys.argv[3]) if len(sys.argv) > 3 else 0x200
funcs, cur = {}, None
for l in open(path).read().split("\n"):
    m = re.search(r"Function : (\S+)", l)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    if cur:
        funcs[cur].append(l)
for name, body in funcs.items():
    if pat not in name:
        continue
    ins = []
    for l in body:
        m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
        if m:
            ins.append((int(m.group(1), 16), m.group(2)))
    print(name, "total", len(ins))
    for addr, txt in ins:
        mm = re.search(r"BRA\S*\s+.*?0x([0-9a-f]+)", txt)
        if "BRA" in txt and mm:
            tgt = int(mm.group(1), 16)
            if tgt < addr and addr - tgt > minb:
                loop = [t for a, t in ins if tgt <= a <= addr]
                c = Counter((t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0] for t in loop)
                print("  loop", hex(tgt), hex(addr), len(loop), c.most_common(24))
