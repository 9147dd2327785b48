#!/bin/bash
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_r02c.txt 2>&1; tail -3 gpurun_out/pytest_gpu_r02c.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()"
timeout 600 python bench.py --steps 50 --warmup 10 > gpurun_out/bench_r02c.json 2> gpurun_out/bench_r02c.err; cut -c1-400 gpurun_out/bench_r02c.json
timeout 600 python scripts/sweep.py --heads > gpurun_out/sweep_heads_r02c.jsonl 2>&1; grep -o '"config": "[^"]*".\{0,120\}' gpurun_out/sweep_heads_r02c.jsonl | head -20
