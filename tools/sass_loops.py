"""Instruction mix of every loop (backward-branch body) in a cuobjdump -sass listing."""
import collections
import re
import sys

lines = open(sys.argv[1]).read().splitlines()
ins = []
for ln in lines:
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/\s+(.*?);", ln)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
addr_idx = {a: i for i, (a, _) in enumerate(ins)}
for i, (a, txt) in enumerate(ins):
    m = re.search(r"BRA\s+(?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", txt)
    if not m or not m.group(1):
        continue
    tgt = int(m.group(1), 16)
    if tgt < a and tgt in addr_idx:
        body = ins[addr_idx[tgt]:i + 1]
        c = collections.Counter()
        for _, t in body:
            op = t.split()
            o = op[1] if op[0].startswith("@") else op[0]
            c[o.split(".")[0]] += 1
        dp = sum(c[k] for k in ("DADD", "DFMA", "DMUL"))
        print(f"loop {tgt:#x}-{a:#x}: {len(body)} instrs, DP={dp}, MUFU={c['MUFU']}, {dict(c.most_common(10))}")
