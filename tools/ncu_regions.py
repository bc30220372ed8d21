"""Summarise an `ncu --page source --csv` dump per kernel launch: share of samples and
instructions between BAR.SYNC boundaries, FFMA share, top stall reasons and hottest lines.
usage: ncu -i x.ncu-rep --page source --csv > src.csv; python tools/ncu_regions.py src.csv [launch] [top]"""
import csv, sys, collections

def f(x):
    try: return float(x)
    except: return 0.0

rows = list(csv.reader(open(sys.argv[1])))
want = int(sys.argv[2]) if len(sys.argv) > 2 else None
top = int(sys.argv[3]) if len(sys.argv) > 3 else 0
starts = [i for i, r in enumerate(rows) if r and r[0] == "Kernel Name"]
seen = 0
for si, s in enumerate(starts):
    e = starts[si + 1] if si + 1 < len(starts) else len(rows)
    hdr = rows[s + 1]
    if "Source" not in hdr: continue
    ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[s + 2:e] if len(r) == len(hdr)]
    if not data or "Instructions Executed" not in ix: continue
    src = [r[ix["Source"]] for r in data]
    if not any("FFMA" in x for x in src): continue   # the SASS view, not the CUDA-C view
    if want is not None and seen != want:
        seen += 1; continue
    seen += 1
    smp = [f(r[ix["# Samples"]]) for r in data]; ins = [f(r[ix["Instructions Executed"]]) for r in data]
    S, I = sum(smp) or 1, sum(ins) or 1
    print(f"== launch {seen-1}: {len(data)} SASS lines, {I:.3g} warp-instr, FFMA {sum(i for i,x in zip(ins,src) if 'FFMA' in x)/I*100:.1f}% of instr")
    bars = [i for i, x in enumerate(src) if "BAR.SYNC" in x]
    prev = 0
    for b in bars + [len(src)]:
        seg = range(prev, min(b + 1, len(src)))
        ss = sum(smp[i] for i in seg); ii = sum(ins[i] for i in seg); ff = sum(ins[i] for i in seg if "FFMA" in src[i])
        print(f"  lines {prev:5d}-{b:5d}: samples {ss/S*100:5.1f}%  instr {ii/I*100:5.1f}%  ffma {ff/I*100:5.1f}%")
        prev = b + 1
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    agg = {c: sum(f(r[ix[c]]) for r in data) for c in cols}
    print("  stalls:", ", ".join(f"{c[6:]} {v/S*100:.1f}%" for c, v in sorted(agg.items(), key=lambda kv: -kv[1])[:7]))
    if top:
        order = sorted(range(len(data)), key=lambda i: -smp[i])[:top]
        for i in sorted(order):
            print(f"    {i:5d} {src[i][:64]:64s} smp {smp[i]/S*100:4.1f}% ins {ins[i]/I*100:4.2f}%")
