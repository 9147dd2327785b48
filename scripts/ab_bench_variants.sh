#!/bin/bash
# Same-box A/B of library variants (lib/variants/libetap_mla_<name>.so) on the headline bench line:
#   bash scripts/ab_bench_variants.sh "" name1 name2 ...   ("" = the product library); 2 rounds each.
#   AB_ARGS="--kv fp8" adds bench.py arguments (same for every variant).
for round in 1 2; do
  for v in "$@"; do
    ETAP_LIB_VARIANT=$v timeout 300 python bench.py $AB_ARGS --steps 100 --warmup 10 --e2e-steps 0 --no-cpu-baseline 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('AB [$v]', round(d['value'],2), round(d['roofline']['kernel_avg_us'],2))"
  done
done
