#!/bin/bash
# ncu captures of the head-group-32 decode kernel (>= 32 heads per GPU) + the head sweep.
# Usage: bash scripts/hg32_profile.sh <tag>
TAG=${1:-r02}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 600 python scripts/sweep.py --heads > gpurun_out/sweep_heads_${TAG}.jsonl 2> gpurun_out/sweep_heads_${TAG}.err
cat gpurun_out/sweep_heads_${TAG}.jsonl
for H in 64 128; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 \
     -o gpurun_out/prof_${TAG}_h${H} python scripts/run_once.py --heads $H --iters 3 > gpurun_out/ncu_${TAG}_h${H}.log 2>&1
  tail -2 gpurun_out/ncu_${TAG}_h${H}.log
done
