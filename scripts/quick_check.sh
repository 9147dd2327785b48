#!/bin/bash
# Quick GPU iteration: GPU tests, step timeline at 1K / 64K, step pieces, one bench line.
timeout 900 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for c in 1024 65536; do CTX=$c timeout 300 python scripts/step_timeline.py 2>&1 | tail -3; done
CTX=65536 timeout 300 python scripts/step_parts.py 2>&1 | tail -7
timeout 600 python bench.py --steps 100 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH', d['value'], d['roofline']['kernel_avg_us'], d['roofline']['frac'])"
[ -n "$AB" ] && env $AB timeout 600 python bench.py --steps 100 --warmup 10 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('BENCH[$AB]', d['value'], d['roofline']['kernel_avg_us'], d['roofline']['frac'])"
