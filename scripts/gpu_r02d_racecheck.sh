# one compute-sanitizer tool per call (B200_PROFILING.md); plain run first
set -x
mkdir -p gpurun_out/sanitizer
python scripts/sanitize_case.py > gpurun_out/sanitizer/plain.log 2>&1 && \
timeout 2400 compute-sanitizer --tool racecheck --racecheck-report hazard --print-limit 50 \
  python scripts/sanitize_case.py > gpurun_out/sanitizer/racecheck.log 2>&1
echo "rc=$?"
tail -5 gpurun_out/sanitizer/racecheck.log
