#!/bin/bash
set -u
O=gpurun_out/r02z
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider -k "low_degree or high_degree" > $O/pytest.log 2>&1; echo "pytest_rc=$?"
tail -4 $O/pytest.log
