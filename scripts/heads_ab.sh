#!/bin/bash
# head-count sweep (16..128 heads at B=16 x 64K) per library variant: bash scripts/heads_ab.sh "" v1 ...
for v in "$@"; do
  echo "== variant '${v:-default}'"
  ETAP_LIB_VARIANT=$v timeout 600 python scripts/sweep.py --heads 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('  ', d['config'], round(min(d['us_per_step_stream'], d['us_per_step_graph']),2))
"
done
