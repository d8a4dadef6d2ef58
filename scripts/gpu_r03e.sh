#!/bin/bash
set -u
O=gpurun_out/r03e
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 1500 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench_rc=$?"
tail -c 600 $O/bench.json; tail -3 $O/bench.err
