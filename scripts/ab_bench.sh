#!/bin/bash
# A/B bench lines: bash scripts/ab_bench.sh "ENV=a" "ENV=b" ...  (empty string = default)
for ab in "$@"; do
  for rep in 1 2; do
    env $ab timeout 600 python bench.py --steps 200 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH[$ab]', round(d['value'],2), round(d['roofline']['kernel_avg_us'],2), round(d['roofline']['frac'],4))"
  done
done
