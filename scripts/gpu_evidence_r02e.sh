#!/bin/bash
# Final round-2 evidence on one B200 (after the CTA-pair kernel): bench lines of both arms (weak N=1,
# strong N=1), launch lists + one ncu capture each of the 16-head K2, the 64-head K2 and the pair K2,
# sweeps (configs, heads, serving, MTP), the pair trace and step timelines.
TAG=${1:-r02e}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,power.limit --format=csv
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --scaling strong --steps 50 --warmup 10 > gpurun_out/bench_strong_${TAG}.json 2> gpurun_out/bench_strong_${TAG}.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
cut -c1-400 gpurun_out/bench_${TAG}.json gpurun_out/bench_strong_${TAG}.json gpurun_out/bench_ref_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_${TAG}.csv python scripts/run_once.py --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG} python scripts/run_once.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_h64_${TAG}.csv python scripts/run_once.py --heads 64 --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_h64_${TAG} python scripts/run_once.py --heads 64 --iters 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_h128_${TAG}.csv python scripts/run_once.py --heads 128 --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pair -s 2 -c 1 -o gpurun_out/prof_h128_${TAG} python scripts/run_once.py --heads 128 --iters 3 > /dev/null 2>&1
ls gpurun_out/*${TAG}*.ncu-rep
timeout 900 python scripts/sweep.py > gpurun_out/sweep_${TAG}.jsonl 2> gpurun_out/sweep_${TAG}.err
timeout 900 python scripts/sweep.py --heads > gpurun_out/sweep_heads_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --serving > gpurun_out/sweep_serving_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 600 python scripts/sweep.py --mtp > gpurun_out/sweep_mtp_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
timeout 300 python scripts/trace_pair.py > gpurun_out/trace_pair_${TAG}.txt 2>&1
(HEADS=128 CTX=65536 timeout 200 python scripts/step_timeline.py; CTX=65536 timeout 200 python scripts/step_timeline.py) > gpurun_out/step_timeline_${TAG}.txt 2>&1
ls -la gpurun_out | tail -5
