"""Warp-stall samples and executed instructions of fk_blur_tma launches by code region.

The line table comes from `nvdisasm -g -c` of the cubin (cuobjdump -xelf all libfovea.so), the
samples from `ncu --page source --csv`; instructions are matched by position in the function.
Regions are the enclosing functions of fk_blur_cols.cu (found by scanning the source), the
kernel body split at its main comment anchors.
usage: python tools/ncu_buckets.py src.csv disasm.txt <function substring> launch [launch ...]"""
import collections, csv, re, sys

SRC = 'paper_2012_08655_b200/csrc/fk_blur_cols.cu'
src_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
launches = [int(x) for x in sys.argv[4:]]
text = open(SRC).read().split('\n')
funcs = []  # (start line, name)
for i, l in enumerate(text, 1):
    m = re.match(r'^(?:__device__ .*?|__global__ .*?)?\b(\w+)\(', l)
    if m and (l.startswith('__device__') or l.startswith('fk_blur')):
        funcs.append((i, m.group(1)))
anchors = []  # inside fk_blur_tma: (line, label)
for i, l in enumerate(text, 1):
    for key, lab in (('mbar_wait(bar + buf, phase)', 'K wait bytes'), ('clamp-to-edge in x (blockwise.py:147): the raw bytes', 'K x patch'),
                     ('horizontal pass (blockwise.py:151): lane = tile row (clamped', 'K H call+ring store'),
                     ('if (lane == 0) mbar_arrive(hbar + buf)', 'K hbar/request'), ('vertical pass (blockwise.py:152) + rounding (convolve.py:15) over the groups', 'K V tasks+out store'),
                     ('Item geometry: g (and r, th, tw', 'K item set-up')):
        if key in l: anchors.append((i, lab))
anchors.sort()
def region(f, ln, op):
    if f != 'fk_blur_cols.cu': return f
    name = None
    for s, n in funcs:
        if s <= ln: name = n
    if name == 'fk_blur_tma':
        lab = 'K prologue/item loop'
        for s, a in anchors:
            if s <= ln and s > 1059: lab = a
        return lab
    if name in ('h_bytes', 'h_float', 'v_task_px'):
        return name + (' FFMA' if 'FFMA' in op else ' other')
    return name or '?'
lines, cur, infn = [], None, False
for l in open(dis):
    if l.startswith('.text.'):
        infn = fn in l; continue
    if not infn: continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if m: cur = (m.group(1).split('/')[-1], int(m.group(2))); continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', l): lines.append(cur)
rows = list(csv.reader(open(src_csv)))
starts = [i for i, r in enumerate(rows) if r and r[0] == 'Kernel Name']
for launch in launches:
    s = starts[launch]; e = starts[launch + 1] if launch + 1 < len(starts) else len(rows)
    hdr = rows[s + 1]; ix = {h: i for i, h in enumerate(hdr)}
    data = [r for r in rows[s + 2:e] if len(r) == len(hdr)]
    if len(data) != len(lines): print(f'!! launch {launch}: {len(data)} SASS rows vs {len(lines)} in the line table')
    S = sum(float(r[ix['# Samples']]) for r in data) or 1
    I = sum(float(r[ix['Instructions Executed']]) for r in data) or 1
    agg = collections.defaultdict(lambda: [0.0, 0.0])
    for i in range(min(len(data), len(lines))):
        f, ln = lines[i] if lines[i] else ('?', 0)
        b = region(f, ln, data[i][ix['Source']])
        agg[b][0] += float(data[i][ix['# Samples']]); agg[b][1] += float(data[i][ix['Instructions Executed']])
    print(f'== launch {launch}: {I:.3g} warp instructions, {S:.0f} samples')
    for b, a in sorted(agg.items(), key=lambda kv: -kv[1][0]):
        if a[0] / S > 0.004 or a[1] / I > 0.004: print(f'  {b:30s} samples {a[0]/S*100:5.1f}%  instr {a[1]/I*100:5.1f}%')
