#!/bin/bash
# Same-box A/B of library variants, interleaved twice (A B A B) against drift:
#   bash scripts/ab_variants.sh "<sweep.py args>" base v1 v2 ...
# ("base" = the in-tree libetap_mla.so; others = lib/variants/libetap_mla_<v>.so)
ARGS=$1; shift
for rep in 1 2; do
  for v in "$@"; do
    if [ "$v" = base ]; then unset ETAP_LIB_VARIANT; else export ETAP_LIB_VARIANT=$v; fi
    echo "== $v (rep $rep) sweep.py $ARGS"
    timeout 600 python scripts/sweep.py $ARGS 2>&1 | grep config | python3 -c "
import sys, json
for l in sys.stdin:
    d = json.loads(l)
    us = d.get('us_per_step', min(d.get('us_per_step_stream', 1e9), d.get('us_per_step_graph20', 1e9)))
    print(f\"  {d['config']:45s} stream {d['us_per_step_stream']:7.1f}  best {us:7.1f}\")"
  done
done
