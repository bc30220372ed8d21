cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out

B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-frames 2 --e2e-steps 1 --no-configs"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -f -o gpurun_out/p_rl $B --width 256 --height 256 --frames 8192 --fixation moving > gpurun_out/p_rl.log 2>&1
tail -2 gpurun_out/p_rl.log
