#!/bin/bash
# k_sus_dc variants (L2 prefetch of the next unit on/off, 2 stages x 10 warps) on C4 / C3,
# parity4 effect on the PUS kernels, then the parity suites.
set -u
O=gpurun_out/r02p
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_nopf.so libgfq_s2w10.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C4 8192 10 sus > $O/kb_c4_$lib.json 2>&1; cut -c1-330 $O/kb_c4_$lib.json
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C3 4096 10 sus > $O/kb_c3_$lib.json 2>&1; cut -c1-330 $O/kb_c3_$lib.json
done
timeout 300 python scripts/kbench.py C5 1024 10 > $O/kb_c5.json 2>&1; cut -c1-700 $O/kb_c5.json
timeout 300 python scripts/kbench.py C4 8192 10 pus > $O/kb_c4_pus.json 2>&1; cut -c1-400 $O/kb_c4_pus.json
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_sync_check.py tests/test_gpu_sus_dc64.py tests/test_gpu_decisions.py -q -x -p no:cacheprovider > $O/pytest.log 2>&1; echo "pytest_rc=$?"
tail -6 $O/pytest.log
du -sh $O
