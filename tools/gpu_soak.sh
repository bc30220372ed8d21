cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
( echo "tools/stress_variants.py 64 5 (default dispatch, fk_blur_cols everywhere, generic kernel, serial class launches; 1080p, random fixations):"; timeout 1200 python tools/stress_variants.py 64 5 | tail -2
  echo; echo "tools/soak.py 300 (random geometries against the generic kernel and the C oracle):"; timeout 1500 python tools/soak.py 300 2>&1 | tail -2
  echo; echo "tools/mixed_check.py 120 (fragments of 4..20 pixels, uint8 and float32: mixed items against the generic kernel and against plans without mixed items):"; timeout 1200 python tools/mixed_check.py 120 | tail -1
  echo; echo "tools/f32_check.py 80 (float32 frames by TMA against the generic kernel):"; timeout 900 python tools/f32_check.py 80 | tail -1 ) > gpurun_out/r02_final_stress.txt 2>&1
cat gpurun_out/r02_final_stress.txt
