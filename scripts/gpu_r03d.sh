#!/bin/bash
set -u
O=gpurun_out/r03d
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1; echo "build_rc=$?"
timeout 600 python bench.py --config C3 --steps 3 --warmup 3 --secondary C1 --conv-frames 256 > $O/bench_c3.json 2> $O/bench_c3.err; echo "bench_rc=$?"
python -c "
import json
b=json.load(open('$O/bench_c3.json'))
print(b['value'], b['schedule_rooflines'], b['secondary']['schedule_rooflines'] if b['secondary'] else None)
print(b['cpu_baseline'])
"
tail -3 $O/bench_c3.err
