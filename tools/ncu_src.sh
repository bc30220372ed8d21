#!/bin/bash
# Source-level counters of one class launch of the headline step (per-SASS executed counts and stall samples):
#   gpurun -- bash tools/ncu_src.sh <launch index, 8 = the 25-47-tap class> [extra bench args]
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
IDX=${1:-8}; shift
ncu --section SourceCounters --section WarpStateStats --clock-control none --import-source on \
    -k regex:fk_blur_tma -s $IDX -c 1 -f -o gpurun_out/src_probe \
    python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs --e2e-frames 2 --e2e-steps 1 "$@" > gpurun_out/src_probe.log 2>&1
ncu -i gpurun_out/src_probe.ncu-rep --page source --csv > gpurun_out/src_probe.csv 2>/dev/null
ls -la gpurun_out/src_probe.*
