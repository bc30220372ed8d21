set -x
cd $GRAFT_REPO_ROOT
timeout 600 python tools/f32_check.py 40 > gpurun_out/f32_check.txt 2>&1; tail -5 gpurun_out/f32_check.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest1.log 2>&1; tail -5 gpurun_out/pytest1.log
for F in 8 16 32 64; do for E in 2.3 1.5; do
timeout 300 python bench.py --dtype f32 --fragment $F --e2 $E --fixation centre --frames 64 --e2e-frames 8 --e2e-steps 1 --steps 5 --warmup 3 --no-cpu-baseline >> gpurun_out/f32_bench1.jsonl 2>>gpurun_out/f32_bench1.err
done; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 2 > gpurun_out/u8_bench1.json 2>gpurun_out/u8_bench1.err
python - <<'PY'
import json
for l in open('gpurun_out/f32_bench1.jsonl'):
    if l.startswith('{'):
        d=json.loads(l); print(d['config']['workload'][:90], round(d['value']), round(d['roofline']['frac'],3))
d=json.loads(open('gpurun_out/u8_bench1.json').read().strip().splitlines()[-1]); print('u8', round(d['value']), round(d['roofline']['frac'],3))
PY
