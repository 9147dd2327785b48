#!/bin/bash
# Pair-kernel evidence on one B200: strong-mode bench line (128 heads), launch list and one ncu capture.
mkdir -p gpurun_out
TAG=r02e
timeout 600 python bench.py --scaling strong --steps 50 --warmup 10 > gpurun_out/bench_strong_${TAG}.json 2> gpurun_out/bench_strong_${TAG}.err; cut -c1-2500 gpurun_out/bench_strong_${TAG}.json; tail -3 gpurun_out/bench_strong_${TAG}.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:etap -s 6 -c 12 --csv --log-file gpurun_out/launches_h128_${TAG}.csv python scripts/run_once.py --heads 128 --iters 7 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:decode_pair -s 2 -c 1 -o gpurun_out/prof_h128_${TAG} python scripts/run_once.py --heads 128 --iters 3 > /dev/null 2>&1
ls gpurun_out/*${TAG}*
