cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest4.log 2>&1; tail -8 gpurun_out/pytest4.log
timeout 300 python tools/bench_stream.py 2000 > gpurun_out/stream.json 2> gpurun_out/stream.err; cat gpurun_out/stream.json; tail -3 gpurun_out/stream.err
