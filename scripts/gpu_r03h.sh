#!/bin/bash
set -u
O=gpurun_out/r03h
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 600 python scripts/kbench.py C5 8192 5 sus > $O/kb_c5_8192.json 2>&1; cut -c1-330 $O/kb_c5_8192.json
timeout 3000 python -m pytest tests -q -m gpu -p no:cacheprovider > $O/pytest_gpu.log 2>&1; echo "pytest_rc=$?"
tail -4 $O/pytest_gpu.log
timeout 300 python __graft_entry__.py smoke > $O/smoke.log 2>&1; echo "smoke_rc=$?"; tail -2 $O/smoke.log
