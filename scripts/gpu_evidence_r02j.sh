#!/bin/bash
# Round-2 final state (fifth session: same kernels as r02i, bench with roofline.read_stream): GPU tests, bench lines (weak,
# strong, FP8, reference arm), ncu of the 16-head K2 with its launch list, the config / head-count
# / serving / MTP sweeps, per-SM handover at 16 and 32 heads.
TAG=${1:-r02j}
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -2
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py --steps 100 --warmup 10 > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
timeout 900 python bench.py --scaling strong --steps 50 --warmup 10 > gpurun_out/bench_strong_${TAG}.json 2> gpurun_out/bench_strong_${TAG}.err
timeout 900 python bench.py --kv fp8 --steps 100 --warmup 10 > gpurun_out/bench_fp8_${TAG}.json 2> gpurun_out/bench_fp8_${TAG}.err
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref_${TAG}.json 2> gpurun_out/bench_ref_${TAG}.err
cut -c1-200 gpurun_out/bench_${TAG}.json gpurun_out/bench_strong_${TAG}.json gpurun_out/bench_fp8_${TAG}.json gpurun_out/bench_ref_${TAG}.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_${TAG}.csv python scripts/run_once.py --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_${TAG} python scripts/run_once.py --iters 3 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_h128_${TAG}.csv python scripts/run_once.py --heads 128 --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pair -s 2 -c 1 -o gpurun_out/prof_h128_${TAG} python scripts/run_once.py --heads 128 --iters 3 > /dev/null 2>&1
timeout 900 python scripts/sweep.py > gpurun_out/sweep_${TAG}.jsonl 2> gpurun_out/sweep_${TAG}.err
timeout 900 python scripts/sweep.py --heads > gpurun_out/sweep_heads_${TAG}.jsonl 2>> gpurun_out/sweep_${TAG}.err
(timeout 120 python scripts/sm_gaps.py; HEADS=32 timeout 120 python scripts/sm_gaps.py) > gpurun_out/sm_gaps_${TAG}.txt 2>&1
ls -la gpurun_out | tail -4
