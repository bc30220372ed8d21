#!/bin/bash
# Everything the round's artefacts are made from, in one gpurun call (B200, one GPU):
#   /usr/local/graft/bin/gpurun --timeout 3000 -- bash tools/final_run.sh r02
# then `tools/collect_profiles.sh r02` here turns gpurun_out/r02_final_* into profiles/.
R=${1:-r02}
O=gpurun_out
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p $O
python -m pytest tests -m gpu -q > $O/${R}_final_pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 > $O/${R}_final_bench.json 2> $O/${R}_final_bench.err
python bench.py --impl reference --steps 2 --warmup 1 > $O/${R}_final_reference.json 2>> $O/${R}_final_bench.err
python tools/bench_stream.py 2000 > $O/${R}_final_stream.json 2>> $O/${R}_final_bench.err
python tools/bench_request.py 2000 > $O/${R}_final_request.json 2>> $O/${R}_final_bench.err
: > $O/${R}_final_exploration.jsonl
X="--steps 5 --warmup 3 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 8"
python bench.py $X --fixation centre >> $O/${R}_final_exploration.jsonl 2>> $O/${R}_final_bench.err
python bench.py $X --fixation corner >> $O/${R}_final_exploration.jsonl 2>> $O/${R}_final_bench.err
python bench.py $X --frames 64 --width 1921 >> $O/${R}_final_exploration.jsonl 2>> $O/${R}_final_bench.err
python bench.py $X --frames 64 --variant 32 --fragment 16 >> $O/${R}_final_exploration.jsonl 2>> $O/${R}_final_bench.err
python bench.py $X --frames 64 --fragment 16 >> $O/${R}_final_exploration.jsonl 2>> $O/${R}_final_bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${R}_final_launches.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-configs --e2e-steps 1 --e2e-frames 8 > /dev/null 2>&1
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs --e2e-frames 2 --e2e-steps 1"
ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -f -o $O/${R}_final_prof_u8 $B > $O/${R}_final_prof_u8.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -f -o $O/${R}_final_prof_f32 $B --dtype f32 --fixation centre --frames 64 --fragment 16 > $O/${R}_final_prof_f32.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -f -o $O/${R}_final_prof_rl $B --width 256 --height 256 --frames 8192 > $O/${R}_final_prof_rl.log 2>&1
tail -3 $O/${R}_final_pytest_gpu.log
ls -la $O/${R}_final_*
