for ctx in 4096 16384 65536; do
  echo "=== fp8 ctx=$ctx"; timeout 300 python scripts/trace_pipeline.py --fp8 --ctx $ctx 2>&1 | tail -40
  echo "=== bf16 ctx=$ctx"; timeout 300 python scripts/trace_pipeline.py --ctx $ctx 2>&1 | tail -12
done
for ctx in 4096 16384; do echo "=== timeline fp8 ctx=$ctx"; FP8=1 CTX=$ctx timeout 300 python scripts/step_timeline.py 2>&1 | tail -20; done
