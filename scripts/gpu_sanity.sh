nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
timeout 1200 python -m pytest tests -q -m gpu 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/bench_r02j.json 2> gpurun_out/bench_r02j.err
timeout 600 python bench.py --scaling strong --steps 50 --warmup 10 > gpurun_out/bench_strong_r02j.json 2> gpurun_out/bench_strong_r02j.err
timeout 600 python bench.py --kv fp8 --steps 100 --warmup 10 > gpurun_out/bench_fp8_r02j.json 2> gpurun_out/bench_fp8_r02j.err
cut -c1-300 gpurun_out/bench_r02j.json gpurun_out/bench_strong_r02j.json gpurun_out/bench_fp8_r02j.json
