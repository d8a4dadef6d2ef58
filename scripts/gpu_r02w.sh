#!/bin/bash
# k_cn_dc (PUS check node by direct convolution, q = 8, 16): parity, then timings against k_cn.
set -u
O=gpurun_out/r02w
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
GFQ_CN_DC=1 timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "(C3 or C4) and PUS" > $O/pytest_cndc.log 2>&1; echo "pytest_cndc_rc=$?"
tail -4 $O/pytest_cndc.log
for v in 0 1; do
  GFQ_CN_DC=$v timeout 300 python scripts/kbench.py C4 8192 10 pus > $O/kb_c4_cndc$v.json 2>&1; cut -c1-420 $O/kb_c4_cndc$v.json
  GFQ_CN_DC=$v timeout 300 python scripts/kbench.py C3 4096 10 pus > $O/kb_c3_cndc$v.json 2>&1; cut -c1-420 $O/kb_c3_cndc$v.json
done
GFQ_CN_DC=1 timeout 900 python -m pytest tests/test_gpu_decisions.py -q -x -p no:cacheprovider -k "(C3 or C4) and pus" > $O/pytest_cndc_dec.log 2>&1; echo "pytest_cndc_dec_rc=$?"
tail -4 $O/pytest_cndc_dec.log
