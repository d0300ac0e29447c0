"""Count fmaheavy-pipe slots per loop iteration from cuobjdump -sass text.

    python tools/sass_slots.py <sass.txt> [start_line end_line]

Weights from tools/probe_*.cu measurements on B200: IMAD.WIDE / IMAD.HI = 2
slots, other IMAD forms = 1, FP64 ops (DFMA, DMUL, DADD, DSETP, DMNMX) = 1 on
the same 64-slot/clk/SM datapath."""
import re
import sys
from collections import Counter

lines = open(sys.argv[1]).read().splitlines()
if len([x for x in sys.argv if not x.startswith('--')]) > 3:
    lines = lines[int(sys.argv[2]) - 1:int(sys.argv[3])]
else:
    # the hot loop: among innermost loops (no backward branch inside), the one
    # carrying the most heavy slots
    loops = []
    for i, l in enumerate(lines):
        m = re.search(r"/\*([0-9a-f]{4,})\*/.*\bBRA(?:\.U)?\s+(?:!?U?P\w+,\s*)?0x([0-9a-f]+)", l)
        if m and int(m.group(2), 16) < int(m.group(1), 16):
            tgt = int(m.group(2), 16)
            i0 = next(k for k, x in enumerate(lines) if re.search(r"/\*0*%x\*/" % tgt, x))
            loops.append((i0, i))
    inner = [(a, b) for a, b in loops if not any(a <= c and d < b and (c, d) != (a, b) for c, d in loops)]

    def weight(span):  # heavy-datapath slots, the weights below
        w = 0
        for l in lines[span[0]:span[1] + 1]:
            mm = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
            if not mm:
                continue
            op = mm.group(1)
            if op.startswith(("IMAD.WIDE", "IMAD.HI")):
                w += 2
            elif op.startswith(("IMAD", "DFMA", "DMUL", "DADD", "DSETP", "DMNMX")):
                w += 1
        return w

    # kernels with a per-instance fast/fallback split (the fused Garner,
    # draw.cuh with_garner) carry two draw loops: the fast one is the lighter
    # of the loops within 60 % of the heaviest ("--lightest"; default heaviest)
    top = max(weight(x) for x in inner)
    if "--lightest" in sys.argv:
        a, b = min((x for x in inner if weight(x) >= 0.6 * top), key=weight)
    else:
        a, b = max(inner, key=weight)
    lines = lines[a:b + 1]
ops = Counter()
heavy = 0.0
alu = 0
total = 0
for l in lines:
    m = re.search(r"\*/\s+(?:@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)", l)
    if not m:
        continue
    op = m.group(1)
    total += 1
    ops[op] += 1
    base = op.split(".")[0]
    if op.startswith("IMAD.WIDE") or op.startswith("IMAD.HI"):
        heavy += 2
    elif base == "IMAD":
        heavy += 1
    elif base in ("DFMA", "DMUL", "DADD", "DSETP", "DMNMX"):
        heavy += 1
    elif base in ("IADD3", "LOP3", "SEL", "ISETP", "SHF", "LEA", "FSEL", "VIADD", "IABS", "PRMT", "MOV", "IMNMX", "VIMNMX"):
        alu += 1
print(f"instructions {total}  heavy slots {heavy}  alu {alu}")
for k, v in ops.most_common():
    print(f"  {v:4d} {k}", flush=True)
