#!/bin/bash
# Same-box A/B of the L2 prefetch depth before the grid dependency (base 2 pages)
# vs 4 and 1 pages (variants hint4, hint1) on the weak (16 heads) and strong (128 heads) bench lines, 3 interleaved reps.
for rep in 1 2 3; do for v in base hint4 hint1; do for mode in weak strong; do
  if [ "$v" = base ]; then unset ETAP_LIB_VARIANT; else export ETAP_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --scaling $mode --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$v $mode', round(d['value'],1))"
done; done; done
