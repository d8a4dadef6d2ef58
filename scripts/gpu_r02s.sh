#!/bin/bash
# k_sus_dc: entries in flight in the streamed variable node (2 / 4 / 8)
set -u
O=gpurun_out/r02s
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_vnu4.so libgfq_vnu8.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C4 8192 10 sus > $O/kb_c4_$lib.json 2>&1; cut -c1-330 $O/kb_c4_$lib.json
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C3 4096 10 sus > $O/kb_c3_$lib.json 2>&1; cut -c1-330 $O/kb_c3_$lib.json
done
