for h in 16 32 128; do echo "== heads $h"; timeout 300 python scripts/trace_pipeline.py --heads $h 2>&1 | head -19; done
