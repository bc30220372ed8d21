#!/bin/bash
# Everything the round's artefacts are made from, in one gpurun call (B200, one GPU):
#   /usr/local/graft/bin/gpurun --timeout 2400 -- bash tools/final_run.sh
# then tools/collect_profiles.sh here turns gpurun_out/r01_final_* into profiles/.
O=gpurun_out
python -m pytest tests -m gpu -q > $O/r01_final_pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 > $O/r01_final_bench.json 2> $O/r01_final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/r01_final_reference.json 2>> $O/r01_final_bench.err
python tools/bench_stream.py 2000 > $O/r01_final_stream.json 2>> $O/r01_final_bench.err
: > $O/r01_final_exploration.jsonl
X="--steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1"
python bench.py $X --frames 32 --e2e-frames 32 --width 3840 --height 2160 --fragment 16 >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
python bench.py $X --frames 8192 --e2e-frames 256 --width 256 --height 256 >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
for F in 8 16 32 64; do
  python bench.py $X --frames 32 --e2e-frames 32 --dtype f32 --fragment $F >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
done
python bench.py $X --frames 32 --e2e-frames 32 --dtype f32 --e2 1.5 >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
python bench.py $X --fixation centre >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
python bench.py $X --fixation corner >> $O/r01_final_exploration.jsonl 2>> $O/r01_final_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/r01_final_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 1 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:fk_blur -c 10 -f -o $O/r01_final_prof \
    python bench.py --frames 32 --steps 1 --warmup 1 --no-cpu-baseline --e2e-steps 1 --e2e-frames 32 > $O/r01_final_prof.log 2>&1
tail -3 $O/r01_final_pytest_gpu.log
