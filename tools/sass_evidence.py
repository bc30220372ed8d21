"""Per kernel of libfovea.so: how many TMA (UTMALDG), mbarrier (SYNCS), cp.async (LDGSTS), FFMA
and PRMT instructions its SASS holds.  usage: python tools/sass_evidence.py > profiles/rNN_sass_tma.txt"""
import collections, re, subprocess
so = "paper_2012_08655_b200/csrc/libfovea.so"
sass = subprocess.run(["cuobjdump", "-sass", so], capture_output=True, text=True).stdout
counts, fn = collections.defaultdict(collections.Counter), None
for line in sass.splitlines():
    m = re.search(r"Function : (\S+)", line)
    if m:
        fn = m.group(1); continue
    m = re.search(r"\b(UTMALDG[.\w]*|SYNCS[.\w]*|LDGSTS[.\w]*|UBLKCP[.\w]*|FFMA|PRMT|BAR\.SYNC[.\w]*)\b", line)
    if m and fn:
        counts[fn][m.group(1)] += 1
names = subprocess.run(["c++filt"], input="\n".join(counts), capture_output=True, text=True).stdout.splitlines()
print(f"# {so}: cuobjdump -sass, instruction counts per kernel (round 2 build)")
for mangled, name in sorted(zip(counts, names), key=lambda x: x[1]):
    short = name.replace("(anonymous namespace)::", "").replace("void ", "", 1)
    short = re.sub(r"\((CUtensorMap_st|fk_|double|float|unsigned|int|const).*", "", short)
    print(f"{short}")
    for op, n in sorted(counts[mangled].items()):
        print(f"    {n:6d}  {op}")
