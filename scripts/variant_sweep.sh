#!/bin/bash
# Sweep (configs 1, 3, 4) for each library variant: bash scripts/variant_sweep.sh "" F1 F2 ...
for v in "$@"; do
  echo "== variant '${v:-default}'"
  ETAP_LIB_VARIANT=$v timeout 600 python scripts/sweep.py --no-config5 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('  ', d['config'], round(min(d['us_per_step_stream'], d['us_per_step_graph']),2))
"
done
