cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest5.log 2>&1; tail -8 gpurun_out/pytest5.log
bash tools/racecheck.sh
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench5.json 2> gpurun_out/bench5.err; tail -3 gpurun_out/bench5.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench5.json').read().strip().splitlines()[-1])
print('headline', round(d['value']), round(d['roofline']['frac'],3), 'e2e', round(d['e2e']['value']), d['clocks'])
for e in d.get('configs') or []:
    print(e['name'], round(e['value']), 'frac', round(e['roofline']['frac'],3), 'ms', round(e['kernel_ms'],3), e.get('request_ms_median'))
PY
