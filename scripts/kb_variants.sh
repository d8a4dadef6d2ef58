#!/bin/bash
# kbench over library variants: kb_variants.sh "C4 C5" lib1 lib2 ...
CFGS=$1; shift
for lib in "$@"; do
  for c in $CFGS; do
    GFQ_LIB_PATH=$PWD/paper_cs_0605069_b200/$lib timeout 300 python scripts/kbench.py $c 1024 20 2>&1 | python -c "
import json,sys
for l in sys.stdin:
  try: r=json.loads(l)
  except Exception: print(l.strip()[:200]); continue
  print('$lib', r['config'], {s:(r[s]['model_GBps'], r[s]['ms_per_iter'], {k:v for k,v in r[s]['per_launch_ms'].items() if k in ('cn','vn','sus')}) for s in ('pus','sus') if s in r})
"
  done
done
