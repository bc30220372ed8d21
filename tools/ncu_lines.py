"""Warp-stall samples of a kernel launch grouped by CUDA source line.

ncu's CSV export of the source page carries SASS only; the line table comes from
`nvdisasm -g -c` of the cubin (cuobjdump -xelf all libfovea.so).  Instructions are matched by
position inside the function.
usage: python tools/ncu_lines.py src.csv disasm.txt <function substring> [launch] [top]"""
import csv, re, sys, collections

src_csv, dis, fn = sys.argv[1], sys.argv[2], sys.argv[3]
launch = int(sys.argv[4]) if len(sys.argv) > 4 else 0
top = int(sys.argv[5]) if len(sys.argv) > 5 else 40
# line table: sequence of (line, inlined-at chain) per instruction of the function
lines, cur, infn = [], None, False
for l in open(dis):
    if l.startswith('.text.'):
        infn = fn in l
        continue
    if not infn: continue
    m = re.match(r'\s*//## File "([^"]+)", line (\d+)(.*)', l)
    if m:
        chain = re.findall(r'line (\d+)', l)
        cur = (m.group(1).split('/')[-1], int(m.group(2)), tuple(int(x) for x in chain[1:]))
        continue
    if re.match(r'\s+/\*[0-9a-f]{4,}\*/\s+\S', l):
        lines.append(cur)
rows = list(csv.reader(open(src_csv)))
starts = [i for i, r in enumerate(rows) if r and r[0] == 'Kernel Name']
s = starts[launch]; e = starts[launch + 1] if launch + 1 < len(starts) else len(rows)
hdr = rows[s + 1]; ix = {h: i for i, h in enumerate(hdr)}
data = [r for r in rows[s + 2:e] if len(r) == len(hdr)]
print(f'launch {launch}: {len(data)} SASS rows, line table {len(lines)} instructions')
n = min(len(data), len(lines))
S = sum(float(r[ix['# Samples']]) for r in data) or 1
I = sum(float(r[ix['Instructions Executed']]) for r in data) or 1
agg = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for i in range(n):
    f, ln, chain = lines[i] if lines[i] else ('?', 0, ())
    # attribute to the outermost line of fk_blur_cols.cu (the kernel body), keep the inner line
    key = (chain[-1] if chain else ln, ln if chain else 0, f)
    a = agg[key]
    a[0] += float(data[i][ix['# Samples']]); a[1] += float(data[i][ix['Instructions Executed']])
    a[2] += float(data[i][ix['Instructions Executed']]) if 'FFMA' in data[i][ix['Source']] else 0
outer = collections.defaultdict(lambda: [0.0, 0.0, 0.0])
for (o, inner, f), a in agg.items():
    for k in range(3): outer[o][k] += a[k]
print('-- by kernel-body line (samples %, instr %, ffma share of its instr)')
for o, a in sorted(outer.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f'  line {o:5d}  samples {a[0]/S*100:5.1f}%  instr {a[1]/I*100:5.1f}%  ffma {a[2]/max(a[1],1)*100:5.1f}%')
