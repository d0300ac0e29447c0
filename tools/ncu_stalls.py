"""Per-opcode warp-stall attribution of the hot loop from an ncu --page source --csv
--print-source sass export (instructions executed >= 1e6).

    ncu -i rep.ncu-rep --page source --csv --print-source sass > src.csv
    python tools/ncu_stalls.py src.csv
"""
import csv, sys, collections, re
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; data = rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
cols = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
# per opcode aggregate of stall samples
agg = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
execs = collections.Counter()
for r in data:
    src = r[ix['Source']].strip()
    m = re.match(r'(@!?U?P\w+\s+)?([A-Z][A-Z0-9_.]*)', src)
    if not m: continue
    op = m.group(2)
    n = int(r[ix['Instructions Executed']] or 0)
    if n < 1000000: continue  # hot loop only
    execs[op] += n
    for c in cols:
        v = int(r[ix[c]] or 0)
        agg[op][c] += v; tot[c] += v
print('total samples by reason:', {k.replace('stall_',''): v for k, v in tot.most_common(10)})
allsum = sum(tot.values())
print('op, execs(M), samples share, top reasons')
for op, c in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:25]:
    s = sum(c.values())
    print(f"{op:22s} {execs[op]/1e6:9.1f} {s/allsum*100:5.1f}%  " + ", ".join(f"{k.replace('stall_','')}={v/s*100:.0f}%" for k, v in c.most_common(4)))
