#!/bin/bash
# A/B of two builds of libfovea.so on a list of bench workloads (one gpurun call):
#   gpurun -- bash tools/ab_run.sh tools/ab/libfovea_base.so [label]
# prints frames/s and the roofline fraction of the tracked build (new) and of the given one (base).
BASE=$1; LABEL=${2:-ab}
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
O=gpurun_out/${LABEL}.txt; : > $O
X="--steps 5 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 8"
run() { # name, args...
  local name=$1; shift
  for which in new base; do
    if [ $which = base ]; then export FK_LIB_PATH=$BASE; else unset FK_LIB_PATH; fi
    python bench.py $X "$@" 2>>gpurun_out/${LABEL}.err | python -c "
import json,sys
for l in sys.stdin:
    l=l.strip()
    if l.startswith('{'):
        d=json.loads(l); print('%-28s %-4s %10.1f frames/s  frac %.3f' % ('$name','$which',d['value'],d['roofline']['frac']))
" >> $O
  done
  unset FK_LIB_PATH
}
run headline
run centre --fixation centre
run u8_F16 --frames 64 --fragment 16
run rl_256 --width 256 --height 256 --frames 8192
run f32_F8 --dtype f32 --fixation centre --frames 64 --fragment 8
run f32_F16 --dtype f32 --fixation centre --frames 64 --fragment 16
run f32_F32 --dtype f32 --fixation centre --frames 64 --fragment 32
run f32_F64 --dtype f32 --fixation centre --frames 64 --fragment 64
run f32_F32_e15 --dtype f32 --fixation centre --frames 64 --fragment 32 --e2 1.5
run 4k_F16 --width 3840 --height 2160 --fragment 16 --frames 16 --fixation centre
cat $O
