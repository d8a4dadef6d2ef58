#!/bin/bash
# Stall-reason captures of the hot kernels (run under gpurun):
#   prof_stalls.sh TAG CONFIG FRAMES SCHEDULE KERNEL_REGEX [SKIP]
# keeps only text summaries in gpurun_out/ (the .ncu-rep stays in /tmp).
set -u
TAG=$1; CFG=$2; NF=$3; SCH=$4; KRE=$5; SKIP=${6:-0}
OUT=gpurun_out/prof_$TAG
mkdir -p $OUT
python scripts/prof_case.py $CFG $NF $SCH 1 > $OUT/case.log 2>&1 || { echo "case failed"; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$KRE" -s $SKIP -c 1 -f -o /tmp/$TAG \
    python scripts/prof_case.py $CFG $NF $SCH 1 > $OUT/ncu.log 2>&1
echo "ncu_rc=$?"
ncu -i /tmp/$TAG.ncu-rep --page raw --csv > /tmp/${TAG}_raw.csv 2>/dev/null
python - /tmp/${TAG}_raw.csv > $OUT/raw_summary.txt <<'PY'
import csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, units, vals = rows[0], rows[1], rows[2:]
keep = ("stall", "dram__bytes", "gpu__time_duration", "sm__inst_executed", "smsp__inst_executed",
        "sm__throughput", "pipe", "l1tex__data_bank", "achieved_occupancy", "registers", "smsp__issue_active",
        "sm__warps_active", "dram__throughput")
for v in vals:
    print("==", v[hdr.index("Kernel Name")][:120])
    for h, u, x in zip(hdr, units, v):
        if any(k in h for k in keep):
            print("%-90s %s %s" % (h, x, u))
PY
python scripts/sass_summary.py /tmp/$TAG.ncu-rep > $OUT/sass_summary.txt 2>&1
ncu -i /tmp/$TAG.ncu-rep --page details --csv > $OUT/details.csv 2>/dev/null
ls -la $OUT
