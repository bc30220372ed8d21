cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python tools/stress_variants.py 150 > gpurun_out/stress.txt 2>&1; tail -3 gpurun_out/stress.txt
timeout 900 python tools/mixed_check.py 30 > gpurun_out/mixed_check.txt 2>&1; tail -2 gpurun_out/mixed_check.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest3.log 2>&1; tail -3 gpurun_out/pytest3.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench3.json 2> gpurun_out/bench3.err; tail -3 gpurun_out/bench3.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench3.json').read().strip().splitlines()[-1])
print('headline', round(d['value']), round(d['roofline']['frac'],3), 'exec/alg', round(d['roofline'].get('executed_over_algorithmic',0),3), 'e2e', round(d['e2e']['value']), d['clocks'])
for e in d.get('configs') or []:
    print(e['name'], round(e['value']), 'frac', round(e['roofline']['frac'],3), 'exec/alg', round(e['roofline'].get('executed_over_algorithmic',0),3), 'ms', round(e['kernel_ms'],3))
PY
