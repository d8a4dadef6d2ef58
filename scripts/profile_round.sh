#!/bin/bash
# Round profiling on one B200 (run under gpurun). Keeps gpurun_out small: ncu
# reports stay in /tmp and only their CSV/JSON summaries come back.
set -u
OUT=gpurun_out
mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench.json 2> $OUT/bench.err; echo "bench_rc=$?"
tail -c 4000 $OUT/bench.json
# per-launch device times of the same command (cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-convergence > $OUT/ncu_launch.log 2>&1
echo "ncu_launch_rc=$?"
# full captures of the hot kernels (same launch size as the bench)
python scripts/prof_case.py C5 8192 1 1 > $OUT/pc.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sus -s 4 -c 1 -f -o /tmp/c5_sus \
    python scripts/prof_case.py C5 8192 1 1 > $OUT/ncu_full.log 2>&1
python scripts/prof_case.py C5 8192 0 1 >> $OUT/pc.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn|k_vn" -c 2 -f -o /tmp/c5_pus \
    python scripts/prof_case.py C5 8192 0 1 >> $OUT/ncu_full.log 2>&1
python scripts/ncu_traffic.py $OUT/ncu_traffic.json C5 /tmp/c5_sus.ncu-rep /tmp/c5_pus.ncu-rep > /dev/null 2>&1
for r in c5_sus c5_pus; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > $OUT/${r}_details.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page source --csv --print-source sass > /tmp/${r}_sass.csv 2>/dev/null
done
ls -la $OUT
