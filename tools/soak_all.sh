cd $GRAFT_REPO_ROOT
X="--steps 5 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 8"
for v in 0 6; do python bench.py $X --variant $v 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('variant $v', round(d['value'],1), round(d['roofline']['frac'],4))
"; done > gpurun_out/nbuf_ab.txt
bash tools/gpu_soak.sh > /dev/null 2>&1
bash tools/racecheck.sh > gpurun_out/racecheck_summary.txt 2>&1
cat gpurun_out/nbuf_ab.txt gpurun_out/r02_final_stress.txt gpurun_out/racecheck_summary.txt
