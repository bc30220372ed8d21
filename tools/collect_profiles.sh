#!/bin/bash
# Turn gpurun_out/<round>_final_* (bench lines, launch list, ncu reports) into the tracked files
# under profiles/.  usage: tools/collect_profiles.sh r02
set -e
R=${1:-r02}
cd "$(dirname "$0")/.."
G=gpurun_out
cp $G/${R}_final_bench.json profiles/${R}_final_bench_n1.json
cp $G/${R}_final_reference.json profiles/${R}_final_reference_arm.json
cp $G/${R}_final_launches.csv profiles/${R}_final_ncu_launches.csv
cp $G/${R}_final_pytest_gpu.log profiles/${R}_final_pytest_gpu.log
cp $G/${R}_final_exploration.jsonl profiles/${R}_final_exploration.jsonl
cp $G/${R}_final_stream.json profiles/${R}_final_stream.json
cp $G/${R}_final_request.json profiles/${R}_final_request.json
# the cubin's line table for the per-region breakdown
rm -rf /tmp/fk_cub && mkdir -p /tmp/fk_cub
( cd /tmp/fk_cub && cuobjdump -xelf all "$OLDPWD/paper_2012_08655_b200/csrc/libfovea.so" > /dev/null && \
  nvdisasm -g -c fk_blur_cols.sm_100a.cubin > cols.dis 2>/dev/null )
for W in u8 f32 rl; do
  ncu -i $G/${R}_final_prof_$W.ncu-rep --page source --csv > $G/${R}f_src_$W.csv 2>/dev/null
  ncu -i $G/${R}_final_prof_$W.ncu-rep --page raw --csv > $G/${R}f_raw_$W.csv 2>/dev/null
  python tools/ncu_brief.py $G/${R}_final_prof_$W.ncu-rep > profiles/${R}_final_ncu_keys_$W.txt
  FN=$([ $W = f32 ] && echo fk_blur_tmaIfLi3 || echo fk_blur_tmaIhLi3)
  python tools/ncu_buckets.py $G/${R}f_src_$W.csv /tmp/fk_cub/cols.dis $FN 2 4 6 8 > profiles/${R}_final_ncu_regions_$W.txt || true
done
python tools/ncu_opmix.py $G/${R}f_src_u8.csv 2 4 6 8 > profiles/${R}_final_ncu_opmix.txt || true
python - "$R" <<'PY'
import csv, json, sys
R = sys.argv[1]
rows = list(csv.reader(open(f'gpurun_out/{R}f_raw_u8.csv')))
hdr = rows[0]
def col(k):
    i = hdr.index(k)
    return [float(r[i]) for r in rows[2:]], rows[1][i]
rd, u1 = col('dram__bytes_read.sum'); wr, u2 = col('dram__bytes_write.sum')
scale = {'Mbyte': 1e6, 'Kbyte': 1e3, 'Gbyte': 1e9, 'byte': 1}
Rd = sum(rd) * scale[u1]; Wb = sum(wr) * scale[u2]
frames = 256  # the capture holds the class launches of one 256-frame step of the headline workload
t = {"source": f"profiles/{R}_final_ncu_keys_u8.txt (ncu --set full, the fk_blur_tma class launches of one "
               "256-frame step of BASELINE configs[1])",
     "frames": frames, "dram_bytes_read": Rd, "dram_bytes_write": Wb,
     "dram_bytes_per_frame": (Rd + Wb) / frames}
json.dump(t, open('profiles/traffic.json', 'w'), indent=1)
print(t)
PY
python tools/sass_evidence.py > profiles/${R}_sass_tma.txt
ls profiles | grep ${R}_
