# compute-sanitizer racecheck on fk_blur_tma with a CTA barrier next to every mbarrier
# (-DFK_DEBUG_CTA_BARRIERS), then memcheck on the shipped build.  Run on the GPU box:
#   gpurun -- 'bash tools/racecheck.sh'
cd ${GRAFT_REPO_ROOT:-.}; mkdir -p gpurun_out
python paper_2012_08655_b200/_build.py --debug-barriers > /dev/null || exit 1
FK_KEEP_BUILD=1 timeout 1500 compute-sanitizer --tool racecheck --racecheck-report all python tools/sanitize_case.py > gpurun_out/racecheck.txt 2>&1
grep -E "RACECHECK SUMMARY|done|Error|hazard" gpurun_out/racecheck.txt | sort | uniq -c | head -20
python paper_2012_08655_b200/_build.py --force > /dev/null
timeout 1500 compute-sanitizer --tool memcheck python tools/sanitize_case.py > gpurun_out/memcheck.txt 2>&1
grep -E "ERROR SUMMARY|done" gpurun_out/memcheck.txt
