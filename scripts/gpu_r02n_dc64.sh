#!/bin/bash
# k_sus_dc64 (q = 64 SUS by direct convolution) against the transform kernel:
# parity gates with the variant on, then kernel timings of both.
set -u
O=gpurun_out/r02n
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
GFQ_SUS_DC64=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -s -p no:cacheprovider -k "C5 and SUS" > $O/pytest_dc64.log 2>&1; echo "pytest_dc64_rc=$?"
grep -E "C5|passed|failed|Error" $O/pytest_dc64.log | tail -12
for v in 0 1; do
  GFQ_SUS_DC64=$v timeout 300 python scripts/kbench.py C5 1024 10 sus > $O/kb_c5_1024_dc$v.json 2>&1; cut -c1-600 $O/kb_c5_1024_dc$v.json
  GFQ_SUS_DC64=$v timeout 600 python scripts/kbench.py C5 8192 5 sus > $O/kb_c5_8192_dc$v.json 2>&1; cut -c1-600 $O/kb_c5_8192_dc$v.json
done
GFQ_SUS_DC64=1 timeout 900 python -m pytest tests/test_gpu_decisions.py -q -x -s -p no:cacheprovider -k "C5" > $O/pytest_dc64_dec.log 2>&1; echo "pytest_dc64_dec_rc=$?"
tail -5 $O/pytest_dc64_dec.log
GFQ_SUS_DC64=1 python scripts/prof_case.py C5 8192 1 1 > $O/pc.log 2>&1 && \
  GFQ_SUS_DC64=1 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_sus -s 4 -c 1 -f -o /tmp/c5_dc64 \
    python scripts/prof_case.py C5 8192 1 1 > $O/ncu_full.log 2>&1
ncu -i /tmp/c5_dc64.ncu-rep --page details --csv > $O/c5_dc64_details.csv 2>/dev/null
python scripts/sass_summary.py /tmp/c5_dc64.ncu-rep > $O/c5_dc64_sass_summary.txt 2>/dev/null
du -sh $O
# small fields through k_sus_dc (GFQ_SUS_DC_MINQ): parity, then timings
GFQ_SUS_DC_MINQ=4 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "(C2 or C3) and SUS" > $O/pytest_dcminq.log 2>&1; echo "pytest_dcminq_rc=$?"
tail -3 $O/pytest_dcminq.log
for v in 16 4; do
  GFQ_SUS_DC_MINQ=$v timeout 300 python scripts/kbench.py C3 4096 10 sus > $O/kb_c3_minq$v.json 2>&1; cut -c1-400 $O/kb_c3_minq$v.json
  GFQ_SUS_DC_MINQ=$v timeout 300 python scripts/kbench.py C2 1024 10 sus > $O/kb_c2_minq$v.json 2>&1; cut -c1-400 $O/kb_c2_minq$v.json
done
du -sh $O
