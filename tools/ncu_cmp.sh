cd $GRAFT_REPO_ROOT
M=gpu__time_duration.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__m_xbar2l1tex_read_bytes.sum,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio,smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio
B="python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-configs --e2e-frames 2 --e2e-steps 1 --dtype f32 --fixation centre --frames 64 --fragment 32"
ncu --metrics $M --clock-control none -k regex:fk_blur_tma -s 4 -c 4 --csv --log-file gpurun_out/cmp_new.csv $B > /dev/null 2>&1
FK_LIB_PATH=tools/ab/libfovea_base.so ncu --metrics $M --clock-control none -k regex:fk_blur_tma -s 4 -c 4 --csv --log-file gpurun_out/cmp_base.csv $B > /dev/null 2>&1
