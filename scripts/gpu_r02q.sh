#!/bin/bash
# Unit-balanced SUS task ranges: kernel timings (C3, C4, C5), W=16 variant of k_sus_dc, SUS parity.
set -u
O=gpurun_out/r02q
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
for lib in libgfq.so libgfq_w16.so; do
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C4 8192 10 sus > $O/kb_c4_$lib.json 2>&1; cut -c1-330 $O/kb_c4_$lib.json
  GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py C3 4096 10 sus > $O/kb_c3_$lib.json 2>&1; cut -c1-330 $O/kb_c3_$lib.json
done
timeout 600 python scripts/kbench.py C5 8192 5 sus > $O/kb_c5_8192.json 2>&1; cut -c1-330 $O/kb_c5_8192.json
timeout 300 python scripts/kbench.py C2 1024 10 sus > $O/kb_c2.json 2>&1; cut -c1-330 $O/kb_c2.json
timeout 300 python scripts/kbench.py C1 64 10 sus > $O/kb_c1.json 2>&1; cut -c1-330 $O/kb_c1.json
timeout 2400 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "SUS or sus or sync or compaction or q256 or q128" > $O/pytest.log 2>&1; echo "pytest_rc=$?"
tail -6 $O/pytest.log
du -sh $O
