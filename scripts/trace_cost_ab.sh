#!/bin/bash
# Cost of the runtime-checked debug stamps: default library vs -DETAP_NO_TRACE (variant notrace)
bash scripts/fp8_ab.sh notrace oldq
bash scripts/variant_sweep.sh "" notrace
for v in "" notrace; do
  echo "== heads variant '${v:-default}'"
  ETAP_LIB_VARIANT=$v timeout 600 python scripts/sweep.py --heads 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: print(l.strip()[:200]); continue
    print('  ', d['config'], round(min(d['us_per_step_stream'], d['us_per_step_graph']),2))
"
done
