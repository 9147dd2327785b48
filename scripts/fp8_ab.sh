#!/bin/bash
# A/B of the FP8 sweep between the default library and variants: bash scripts/fp8_ab.sh V1 V2 ...
for rep in 1 2; do
for v in "" "$@"; do
  echo "== variant '${v:-default}' rep $rep"
  ETAP_LIB_VARIANT=$v timeout 600 python scripts/sweep.py --fp8 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('  ', d['config'], round(d['us_per_step_stream'],2))
"
done
done
