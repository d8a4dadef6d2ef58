#!/bin/bash
# Round-2 measurement pass on one B200 (under gpurun): new-feature tests first,
# then bench, launch list, full ncu captures of the hot kernels (summaries only:
# gpurun_out must stay under 64 MiB), then the whole GPU suite.
set -u
O=gpurun_out/r03c
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 300 python scripts/kbench_q256.py 512 5 > $O/kb_q256.json 2>&1; cut -c1-500 $O/kb_q256.json
timeout 300 python scripts/kbench.py X7 1024 10 > $O/kb_x7.json 2>&1; cut -c1-200 $O/kb_x7.json
for c in C1 C2 C3; do timeout 300 python scripts/kbench.py $c $(python -c "import synth;print(synth.CONFIGS['$c'].frames)") 10 > $O/kb_$c.json 2>&1; done
timeout 1500 python bench.py --steps 3 --warmup 3 > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"
tail -c 1500 $O/bench.json; tail -3 $O/bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches.csv \
    python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-convergence --secondary '' > $O/ncu_launch.log 2>&1
echo "ncu_launch_rc=$?"
python scripts/launch_summary.py $O/launches.csv $O/launch_summary.json > /dev/null 2>&1
gzip -f $O/launches.csv
python scripts/prof_case.py C5 8192 1 1 > $O/pc.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sus -s 4 -c 1 -f -o /tmp/c5_sus \
    python scripts/prof_case.py C5 8192 1 1 > $O/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn|k_vn" -c 2 -f -o /tmp/c5_pus \
    python scripts/prof_case.py C5 8192 0 1 >> $O/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sus -s 4 -c 1 -f -o /tmp/c4_sus \
    python scripts/prof_case.py C4 8192 1 1 >> $O/ncu_full.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cn|k_vn" -c 2 -f -o /tmp/c4_pus \
    python scripts/prof_case.py C4 8192 0 1 >> $O/ncu_full.log 2>&1
python scripts/ncu_traffic.py $O/ncu_traffic_c5.json C5 /tmp/c5_sus.ncu-rep /tmp/c5_pus.ncu-rep > /dev/null 2>&1
python scripts/ncu_traffic.py $O/ncu_traffic_c4.json C4 /tmp/c4_sus.ncu-rep /tmp/c4_pus.ncu-rep > /dev/null 2>&1
for r in c5_sus c5_pus c4_sus c4_pus; do
  ncu -i /tmp/$r.ncu-rep --page details --csv > $O/${r}_details.csv 2>/dev/null
  ncu -i /tmp/$r.ncu-rep --page raw --csv > $O/${r}_raw.csv 2>/dev/null
  python scripts/sass_summary.py /tmp/$r.ncu-rep > $O/${r}_sass_summary.txt 2>/dev/null
done
du -sh $O
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -8 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke_rc=$?"; tail -3 $O/smoke.log
du -sh $O
