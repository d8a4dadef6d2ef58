#!/bin/bash
# k_sus_dc warps per CTA for q = 8 (32 / 24 / 16), q = 16 at 16 warps, work-balanced k_vn (C4, C5 PUS).
set -u
O=gpurun_out/r02r
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_w8_24.so libgfq_w8_16.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C3 4096 10 sus > $O/kb_c3_$lib.json 2>&1; cut -c1-330 $O/kb_c3_$lib.json
done
timeout 300 python scripts/kbench.py C4 8192 10 > $O/kb_c4.json 2>&1; cut -c1-900 $O/kb_c4.json
timeout 300 python scripts/kbench.py C5 1024 10 pus > $O/kb_c5_1024.json 2>&1; cut -c1-500 $O/kb_c5_1024.json
timeout 600 python scripts/kbench.py C5 5120 5 pus > $O/kb_c5_5120.json 2>&1; cut -c1-500 $O/kb_c5_5120.json
timeout 300 python scripts/kbench.py C3 4096 10 pus > $O/kb_c3_pus.json 2>&1; cut -c1-500 $O/kb_c3_pus.json
timeout 300 python scripts/kbench.py C2 1024 10 > $O/kb_c2.json 2>&1; cut -c1-900 $O/kb_c2.json
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest_rc=$?"
tail -3 $O/pytest.log
