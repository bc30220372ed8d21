# ncu captures of the blur kernels on three workloads (one step each after warm-up)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --e2e-frames 2 --e2e-steps 1"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -o gpurun_out/p_u8 $B > gpurun_out/p_u8.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 3 -c 3 -o gpurun_out/p_f32 $B --dtype f32 --fixation centre --frames 64 > gpurun_out/p_f32.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fk_blur_tma -s 5 -c 5 -o gpurun_out/p_rl $B --width 256 --height 256 --frames 8192 > gpurun_out/p_rl.log 2>&1
ls -la gpurun_out/*.ncu-rep
