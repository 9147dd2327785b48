#!/bin/bash
# Full measurement round: gpu_round.sh (smoke, tests, bench both arms, launch list, ncu of K2),
# the config sweeps (bf16, heads, MTP, FP8) and an ncu capture of the FP8 kernel.
TAG=${1:-r01}
bash scripts/gpu_round.sh $TAG
timeout 900 python scripts/sweep.py > gpurun_out/sweep_${TAG}.jsonl 2>&1
timeout 600 python scripts/sweep.py --heads >> gpurun_out/sweep_${TAG}.jsonl 2>&1
timeout 600 python scripts/sweep.py --mtp >> gpurun_out/sweep_${TAG}.jsonl 2>&1
timeout 900 python scripts/sweep.py --fp8 --heads >> gpurun_out/sweep_${TAG}.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fp8 -s 2 -c 1 -o gpurun_out/prof_fp8_${TAG} python scripts/run_once.py --fp8 --iters 3 > gpurun_out/ncu_fp8_${TAG}.log 2>&1
tail -n 2 gpurun_out/ncu_fp8_${TAG}.log
