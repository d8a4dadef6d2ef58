#!/bin/bash
# Dedicated producer warp for the 8-warp groups (q = 64, 128): k_cn / k_vn / k_sus timings.
set -u
O=gpurun_out/r02v
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_pw8.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C5 1024 10 > $O/kb_c5_1024_$lib.json 2>&1; cut -c1-900 $O/kb_c5_1024_$lib.json
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 600 python scripts/kbench.py C5 8192 5 sus > $O/kb_c5_8192_$lib.json 2>&1; cut -c1-330 $O/kb_c5_8192_$lib.json
done
