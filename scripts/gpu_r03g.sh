#!/bin/bash
set -u
O=gpurun_out/r03g
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 300 python scripts/kbench.py C5 1024 10 sus > $O/kb_c5_1024.json 2>&1; echo "kb_rc=$?"; cut -c1-330 $O/kb_c5_1024.json
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "C5 and SUS" > $O/pytest_c5.log 2>&1; echo "pytest_c5_rc=$?"; tail -3 $O/pytest_c5.log
timeout 600 python scripts/kbench.py C5 8192 5 sus > $O/kb_c5_8192.json 2>&1; cut -c1-330 $O/kb_c5_8192.json
timeout 300 python scripts/kbench.py X7 1024 10 sus > $O/kb_x7.json 2>&1; cut -c1-330 $O/kb_x7.json
timeout 2400 python -m pytest tests -q -x -m gpu -p no:cacheprovider -k "SUS or sus or sync or q128 or compaction or decisions" > $O/pytest.log 2>&1; echo "pytest_rc=$?"
tail -4 $O/pytest.log
