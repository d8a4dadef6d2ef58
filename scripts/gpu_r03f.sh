#!/bin/bash
set -u
O=gpurun_out/r03f
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
python scripts/prof_case.py C5 8192 1 1 > $O/pc.log 2>&1 && \
  timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sus -s 4 -c 1 -f -o /tmp/c5_sus \
    python scripts/prof_case.py C5 8192 1 1 > $O/ncu_full.log 2>&1
python scripts/sass_export.py /tmp/c5_sus.ncu-rep $O/c5_sus_sass.csv > $O/export.log 2>&1
head -3 $O/export.log | cut -c1-600; wc -l $O/c5_sus_sass.csv; head -5 $O/c5_sus_sass.csv
gzip -f $O/c5_sus_sass.csv
