for rep in 1 2 3; do for v in base cpair1 cpair2; do
  if [ "$v" = base ]; then unset ETAP_LIB_VARIANT; else export ETAP_LIB_VARIANT=$v; fi
  timeout 300 python bench.py --scaling strong --steps 50 --warmup 10 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
  python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); print('$v', round(d['value'],1), round(d['roofline']['kernel_avg_us'],1))"
done; done
