bash scripts/variant_sweep.sh "" h0 h3 h4 "" h0 h3 h4
for v in "" h3 h4; do echo "== serving '$v'"; ETAP_LIB_VARIANT=$v timeout 300 python scripts/sweep.py --serving | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('  ', d['config'], round(d['us_per_step_stream'],2))"; done
