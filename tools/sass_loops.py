"""List the backward branches (loops) of a cuobjdump -sass listing with their
body length in instructions and the opcode mix of each body:
  python tools/sass_loops.py file.sass [min_len]"""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
minlen = int(sys.argv[2]) if len(sys.argv) > 2 else 40
ins = []
for l in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA (?:\S+, )?0x([0-9a-f]+)", txt)
    if not m:
        continue
    t = int(m.group(1), 16)
    if t < a and t in addr_idx:
        body = ins[addr_idx[t]:i + 1]
        if len(body) < minlen:
            continue
        ops = Counter()
        for _, x in body:
            x = re.sub(r"^@!?U?P\w+\s+", "", x)
            ops[x.split()[0].split(".")[0]] += 1
        print(f"loop {t:#x}..{a:#x}: {len(body)} instrs  " +
              " ".join(f"{k}:{v}" for k, v in ops.most_common(14)))
