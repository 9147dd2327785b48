#!/bin/bash
# A/B of the schedule read before the grid dependency (default) vs after it (ETAP_EARLY_META=0):
# step timeline at 1K / 64K, the config sweep, serving mixes and FP8, each arm on the same box.
mkdir -p gpurun_out
for c in 1024 65536; do CTX=$c timeout 200 python scripts/step_timeline.py 2>&1 | tail -2; done
for arm in 1 0; do
  echo "== ETAP_EARLY_META=$arm"
  ETAP_EARLY_META=$arm timeout 900 python scripts/sweep.py --no-config5 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config']:40s} stream {d['us_per_step_stream']:8.2f} graph {d['us_per_step_graph']:8.2f}\")"
  ETAP_EARLY_META=$arm timeout 900 python scripts/sweep.py --serving 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config']:40s} stream {d['us_per_step_stream']:8.2f} graph {d['us_per_step_graph']:8.2f}\")"
  ETAP_EARLY_META=$arm timeout 900 python scripts/sweep.py --fp8 2>&1 | python -c "
import json,sys
for l in sys.stdin:
    try: d=json.loads(l)
    except Exception: continue
    print(f\"{d['config']:40s} stream {d['us_per_step_stream']:8.2f}\")"
  ETAP_EARLY_META=$arm timeout 600 python bench.py --steps 100 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['roofline']['kernel_avg_us'], d['roofline']['frac'])"
done
