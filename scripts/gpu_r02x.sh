#!/bin/bash
set -u
O=gpurun_out/r02x
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_cn_s2.so libgfq_cn_s3.so; do
  GFQ_CN_DC=1 GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C4 8192 10 pus > $O/kb_c4_$lib.json 2>&1; cut -c1-420 $O/kb_c4_$lib.json | grep -o '"lib[^,]*\|"cn": [0-9.]*\|model_GBps": [0-9.]*'
  GFQ_CN_DC=1 GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C3 4096 10 pus > $O/kb_c3_$lib.json 2>&1; cut -c1-420 $O/kb_c3_$lib.json | grep -o '"lib[^,]*\|"cn": [0-9.]*\|model_GBps": [0-9.]*'
done
