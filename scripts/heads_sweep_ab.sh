#!/bin/bash
# Same-box A/B of library variants on the head-count sweep: bash scripts/heads_sweep_ab.sh v1 v2 ...
# ("base" = the in-tree libetap_mla.so; others = lib/variants/libetap_mla_<v>.so)
for v in "$@"; do
  if [ "$v" = base ]; then unset ETAP_LIB_VARIANT; else export ETAP_LIB_VARIANT=$v; fi
  echo "== $v"
  timeout 600 python scripts/sweep.py --heads 2>&1 | grep config | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l); print(f\"  {d['config']:45s} stream {d['us_per_step_stream']:7.1f}  graph20 {d['us_per_step_graph20']:7.1f}\")"
done
