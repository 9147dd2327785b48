timeout 900 python -m pytest tests -q -m gpu 2>&1 | tail -3
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
timeout 300 python scripts/sweep.py --fp8
timeout 300 python scripts/trace_cta.py --fp8 --ctx 16384 2>&1 | head -12
