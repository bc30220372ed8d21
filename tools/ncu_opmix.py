"""Instruction mix by opcode of each profiled launch (from `ncu --page source --csv`).
usage: python tools/ncu_opmix.py src.csv [launch ...]"""
import csv, collections, re, sys

def f(x):
    try: return float(x)
    except ValueError: return 0.0

rows = list(csv.reader(open(sys.argv[1])))
want = [int(x) for x in sys.argv[2:]]
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
seen = -1
for si, s in enumerate(starts):
    e = starts[si + 1] if si + 1 < len(starts) else len(rows)
    hdr = rows[s + 1]
    if "Source" not in hdr: continue
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[s + 2:e] if len(r) == len(hdr)]
    src = [r[ix["Source"]] for r in data]
    if not any("FFMA" in x for x in src): continue
    seen += 1
    if want and seen not in want: continue
    ops = collections.Counter(); smp = collections.Counter()
    for r in data:
        m = re.match(r'\s*(@!?U?P\d+\s+)?([A-Z0-9_]+(\.[A-Z0-9_]+)*)', r[ix["Source"]])
        full = m.group(2) if m else '?'
        op = full.split('.')[0]
        if op in ('LDS', 'STS', 'LDG', 'STG', 'F2I', 'I2F', 'I2FP', 'F2FP', 'LDGSTS'): op = full
        ops[op] += f(r[ix["Instructions Executed"]]); smp[op] += f(r[ix["# Samples"]])
    I = sum(ops.values()) or 1; S = sum(smp.values()) or 1
    print(f"== launch {seen}: {I:.3g} warp-instr")
    for k, v in ops.most_common(30):
        print(f"  {k:24s} instr {v/I*100:5.2f}%  samples {smp[k]/S*100:5.2f}%")
