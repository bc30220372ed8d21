#!/bin/bash
# strip-height cap (FK_STRIP_ROWS_FORCE) against batch size on 1080p uint8, moving fixation: what fk_strip_rows_for encodes
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
O=gpurun_out/strip_sweep.txt; : > $O
X="--steps 5 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 2"
for N in 1 4 8 16 32 64; do for S in 32 64 128 256 512 1024; do
  FK_STRIP_ROWS_FORCE=$S python bench.py $X --frames $N 2>/dev/null | python -c "
import json,sys
for l in sys.stdin:
    if l.startswith('{'):
        d=json.loads(l); print('frames %3d strip %4d  %9.1f frames/s  frac %.3f' % ($N,$S,d['value'],d['roofline']['frac']))
" >> $O
done; done
cat $O
