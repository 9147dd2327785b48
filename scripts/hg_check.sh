set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -x -q -m gpu 2>&1 | tail -15
timeout 600 python scripts/sweep.py --heads 2>&1 | tail -6
ETAP_GROUP_LANES=0 timeout 600 python scripts/sweep.py --heads 2>&1 | tail -6
