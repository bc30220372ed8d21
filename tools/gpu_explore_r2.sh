cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
./tools/ubench_pattern.bin > gpurun_out/r02_ubench_pattern.txt 2>&1
./tools/ubench_vloop.bin > gpurun_out/r02_ubench_vloop.txt 2>&1
./tools/proto_ffma2.bin > gpurun_out/r02_proto_loops.txt 2>&1
tail -3 gpurun_out/r02_proto_loops.txt
