#!/bin/bash
# bench workloads under a list of environment settings (experiments): gpurun -- bash tools/ab_env.sh label
LABEL=${1:-abenv}
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
O=gpurun_out/${LABEL}.txt; : > $O
X="--steps 5 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 8"
run() { # name, env, args...
  local name=$1; local envs=$2; shift; shift
  env $envs python bench.py $X "$@" 2>>gpurun_out/${LABEL}.err | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('%-14s %-40s %10.1f frames/s  frac %.3f' % ('$name','$envs',d['value'],d['roofline']['frac']))
" >> $O
}
for E in ${ENVS:-"FK_X=0"}; do
  run f32_F16 "$E" --dtype f32 --fixation centre --frames 64 --fragment 16
  run f32_F32 "$E" --dtype f32 --fixation centre --frames 64 --fragment 32
  run f32_F32_e15 "$E" --dtype f32 --fixation centre --frames 64 --fragment 32 --e2 1.5
  run f32_F64 "$E" --dtype f32 --fixation centre --frames 64 --fragment 64
  run f32_F8 "$E" --dtype f32 --fixation centre --frames 64 --fragment 8
  run headline "$E"
  run centre "$E" --fixation centre
  run rl_256 "$E" --width 256 --height 256 --frames 8192
  run 4k_F16 "$E" --width 3840 --height 2160 --fragment 16 --frames 16 --fixation centre
done
cat $O
