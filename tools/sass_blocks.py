"""Opcode histogram per basic block of a cuobjdump -sass listing (blocks split at branch
targets); prints the blocks holding MUFU.EX2 — the softmax loop bodies."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for l in lines:
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', l)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
targets = set()
for _, t in ins:
    for m in re.finditer(r'(?:BRA|BRX|JMP|CALL|WARPSYNC|BSSY)[^`]*`\(\.L_x_\d+\)|0x([0-9a-f]+)', t):
        pass
for _, t in ins:
    m = re.search(r'\b(?:BRA|BSSY\S*\s+\S+,)\s.*?0x([0-9a-f]+)', t)
    if m:
        targets.add(int(m.group(1), 16))
blocks, cur, start = [], [], ins[0][0]
for a, t in ins:
    if a in targets and cur:
        blocks.append((start, cur)); cur = []; start = a
    cur.append(t)
    if re.search(r'\b(BRA|EXIT|RET)\b', t):
        blocks.append((start, cur)); cur = []; start = None
        start = a + 16
blocks.append((start, cur))
minmufu = int(sys.argv[2]) if len(sys.argv) > 2 else 16
for s, b in blocks:
    ops = []
    for t in b:
        t = re.sub(r'^@!?U?P[T0-9]+\s+', '', t)
        ops.append(t.split()[0])
    c = collections.Counter(o.split('.')[0] for o in ops)
    if c['MUFU'] >= minmufu:
        print(hex(s), len(b), sorted(c.items(), key=lambda t: -t[1]))
        print('   full ops:', sorted(collections.Counter(ops).items(), key=lambda t: -t[1])[:40])
