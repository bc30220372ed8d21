#!/bin/bash
# Turn gpurun_out/r01_final_* (bench lines, launch list, ncu report) into the tracked files
# under profiles/.  usage: tools/collect_profiles.sh
set -e
cd "$(dirname "$0")/.."
( cd gpurun_out && ncu -i r01_final_prof.ncu-rep --page source --csv > r01f_src.csv 2>/dev/null; \
  ncu -i r01_final_prof.ncu-rep --page raw --csv > r01f_raw.csv 2>/dev/null )
python tools/ncu_keys.py gpurun_out/r01f_raw.csv > profiles/r01_final_ncu_keys.txt
python tools/ncu_regions.py gpurun_out/r01f_src.csv > profiles/r01_final_ncu_regions.txt
python tools/ncu_opmix.py gpurun_out/r01f_src.csv 2 4 6 8 > profiles/r01_final_ncu_opmix.txt
cp gpurun_out/r01_final_bench.json profiles/r01_final_bench_n1.json
cp gpurun_out/r01_final_reference.json profiles/r01_final_reference_arm.json
cp gpurun_out/r01_final_launches.csv profiles/r01_final_ncu_launches.csv
cp gpurun_out/r01_final_pytest_gpu.log profiles/r01_final_pytest_gpu.log
cp gpurun_out/r01_final_exploration.jsonl profiles/r01_final_exploration.jsonl
cp gpurun_out/r01_final_stream.json profiles/r01_final_stream.json
python - <<'PY'
import csv, json
rows = list(csv.reader(open('gpurun_out/r01f_raw.csv')))
hdr = rows[0]
def col(k):
    i = hdr.index(k)
    return [float(r[i]) for r in rows[2:]], rows[1][i]
rd, u1 = col('dram__bytes_read.sum'); wr, u2 = col('dram__bytes_write.sum')
scale = {'Mbyte': 1e6, 'Kbyte': 1e3, 'Gbyte': 1e9, 'byte': 1}
R = sum(rd) * scale[u1]; Wb = sum(wr) * scale[u2]
steps = 2  # the capture holds the class launches of two 32-frame steps
t = {"source": "profiles/r01_final_ncu_keys.txt (ncu --set full, 32-frame batch, the "
               "fk_blur_bytes class launches of two steps)",
     "frames": 32 * steps, "dram_bytes_read": R, "dram_bytes_write": Wb,
     "dram_bytes_per_frame": (R + Wb) / (32 * steps)}
json.dump(t, open('profiles/traffic.json', 'w'), indent=1)
print(t)
PY
