set -x
timeout 300 python scripts/trace_pipeline.py --heads 128 2>&1 | tail -40 > gpurun_out/trace_h128.txt
timeout 300 python scripts/trace_pipeline.py --heads 16 2>&1 | tail -40 > gpurun_out/trace_h16.txt
timeout 300 python scripts/trace_pipeline.py --heads 64 2>&1 | tail -40 > gpurun_out/trace_h64.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_fp8 -s 2 -c 1 -o gpurun_out/prof_fp8 python scripts/run_once.py --fp8 --iters 3 > gpurun_out/ncu_fp8.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:decode_kernel -s 2 -c 1 -o gpurun_out/prof_h128 python scripts/run_once.py --heads 128 --iters 3 > gpurun_out/ncu_h128.log 2>&1
tail -2 gpurun_out/ncu_fp8.log gpurun_out/ncu_h128.log
