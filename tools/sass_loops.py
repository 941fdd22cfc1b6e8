"""List backward branches (loops) in a SASS listing from tools/sass_section.py:
loop body size, MUFU count and an opcode histogram."""
import collections
import re
import sys

lines = [l.split(" ", 1) for l in open(sys.argv[1]).read().splitlines() if " " in l]
addr = [int(a, 16) for a, _ in lines]
idx = {a: i for i, a in enumerate(addr)}
min_mufu = int(sys.argv[2]) if len(sys.argv) > 2 else 1
for i, (a, ins) in enumerate(lines):
    m = re.search(r"BRA\s+(?:`\()?.*?0x([0-9a-f]+)", ins)
    if not m:
        continue
    tgt = int(m.group(1), 16)
    if tgt >= addr[i] or tgt not in idx:
        continue
    body = [x for _, x in lines[idx[tgt]:i + 1]]
    ops = collections.Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for x in body)
    if ops["MUFU"] < min_mufu:
        continue
    print(f"loop {tgt:x}-{addr[i]:x}: {len(body)} instr, MUFU {ops['MUFU']}")
    print("   ", dict(ops.most_common(18)))
