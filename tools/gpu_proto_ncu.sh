cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for cfg in "53 2 0" "53 1 0" "53 2 1" "53 1 1"; do
  n=$(echo $cfg | tr ' ' '_')
  timeout 300 ncu --set full --clock-control none --import-source on -c 1 -f -o gpurun_out/proto_$n ./tools/proto_ffma2.bin $cfg > gpurun_out/proto_$n.log 2>&1
done
ls -la gpurun_out/*.ncu-rep
