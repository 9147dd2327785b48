#!/bin/bash
# Round-2 evidence session on one B200: sanitizer, streaming bound, launch lists + ncu of the
# 16-head K2, the FP8 K2 and the 64/128-head K2, the reference harness, sweeps, bench lines.
TAG=${1:-r02d}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
bash scripts/gpu_call_sanitize.sh
timeout 300 python scripts/stream_bench.py > gpurun_out/stream_bench_${TAG}.txt 2>&1; cat gpurun_out/stream_bench_${TAG}.txt
# launch lists (cold, serialised) and one full capture per kernel
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_${TAG}.csv python scripts/run_once.py --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG} python scripts/run_once.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_fp8_${TAG}.csv python scripts/run_once.py --fp8 --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_fp8 -s 2 -c 1 -o gpurun_out/prof_fp8_${TAG} python scripts/run_once.py --fp8 --iters 3 > /dev/null 2>&1
for H in 64 128; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_h${H}_${TAG}.csv python scripts/run_once.py --heads $H --iters 7 > /dev/null 2>&1
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_h${H}_${TAG} python scripts/run_once.py --heads $H --iters 3 > /dev/null 2>&1
done
ls gpurun_out/*.ncu-rep
# the reference's own harness with the etap_b200 mode + the integration binary
timeout 900 oracle/_ref/etaplab_harness bench 1024 4096 16384 > gpurun_out/harness_bench_${TAG}.csv 2> gpurun_out/harness_bench_${TAG}.err; cat gpurun_out/harness_bench_${TAG}.csv
timeout 900 oracle/_ref/etaplab_harness verify 1e-4 > gpurun_out/harness_verify_${TAG}.txt 2>&1; echo "verify rc=$?" >> gpurun_out/harness_verify_${TAG}.txt; tail -2 gpurun_out/harness_verify_${TAG}.txt
timeout 900 oracle/_ref/etaplab_harness verify 1e-4 corrupt > gpurun_out/harness_verify_corrupt_${TAG}.txt 2>&1; echo "verify rc=$?" >> gpurun_out/harness_verify_corrupt_${TAG}.txt; tail -2 gpurun_out/harness_verify_corrupt_${TAG}.txt
timeout 900 oracle/_ref/etaplab_b200_integration > gpurun_out/integration_${TAG}.jsonl 2>&1; echo "rc=$?"
# sweeps
timeout 900 python scripts/sweep.py > gpurun_out/sweep_${TAG}.jsonl 2> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --heads > gpurun_out/sweep_heads_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --fp8 --heads > gpurun_out/sweep_fp8_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --mtp > gpurun_out/sweep_mtp_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --serving > gpurun_out/sweep_serving_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
# bench lines: reference arm, weak N=1, strong N=1
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --scaling strong --steps 50 --warmup 10 > gpurun_out/bench_strong_${TAG}.json 2> gpurun_out/bench_strong_${TAG}.err
cat gpurun_out/bench_${TAG}.json gpurun_out/bench_strong_${TAG}.json | cut -c1-600
# round-2 continuation probes
timeout 600 python scripts/orientation_claim.py > gpurun_out/orientation_${TAG}.jsonl 2>&1
timeout 300 python scripts/tail_spread.py > gpurun_out/tail_spread_${TAG}.txt 2>&1
for H in 16 64 128; do echo "== heads $H"; timeout 300 python scripts/trace_pipeline.py --heads $H 2>&1 | head -21; done > gpurun_out/trace_${TAG}.txt 2>&1
ls -la gpurun_out | tail -5
