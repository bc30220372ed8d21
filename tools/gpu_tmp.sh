cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest7.log 2>&1; tail -3 gpurun_out/pytest7.log
timeout 600 python tools/mixed_check.py 20 | tail -1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench7.json 2> gpurun_out/bench7.err; tail -3 gpurun_out/bench7.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench7.json').read().strip().splitlines()[-1])
print('headline', round(d['value']), round(d['roofline']['frac'],4), 'kernel', d['roofline']['kernel_ms'], 'e2e', round(d['e2e']['value']))
for e in d.get('configs') or []:
    print(e['name'], round(e['value']), 'frac', round(e['roofline']['frac'],3), 'ms', round(e['ms_per_step'],3), 'kernel', round(e['kernel_ms'],3), e.get('request_ms_median'))
PY
