#!/bin/bash
# New compaction tests + multi-GPU guard on a 1-GPU box.
set -u
O=gpurun_out/r02u
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 1200 python -m pytest tests/test_gpu_compaction.py -q -x -p no:cacheprovider > $O/pytest_compaction.log 2>&1; echo "pytest_rc=$?"
tail -4 $O/pytest_compaction.log
timeout 300 python bench.py --gpus 2 --steps 1 --warmup 3 > $O/bench_gpus2.log 2>&1; echo "bench_gpus2_rc=$?"
tail -5 $O/bench_gpus2.log | cut -c1-300
