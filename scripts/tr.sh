timeout 600 python -m pytest tests -x -q -m gpu 2>&1 | tail -3
for h in 16 32 128; do echo "== heads $h"; timeout 300 python scripts/trace_pipeline.py --heads $h 2>&1 | head -20; done
