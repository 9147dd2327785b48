#!/bin/bash
# Stream launches vs 20-step CUDA graphs, with and without programmatic dependent launch (ETAP_PDL).
for pdl in 1 0; do
ETAP_PDL=$pdl timeout 900 python - <<'PY'
import os, sys, json
sys.path.insert(0, os.getcwd())
import importlib.util
spec = importlib.util.spec_from_file_location("sweep", "scripts/sweep.py"); m = importlib.util.module_from_spec(spec); spec.loader.exec_module(m)
from paper_2506_01969_b200 import inputs
import io, contextlib
for seqlens, heads, label in (([1024] * 16, 16, "B16x1K"), ([65536] * 16, 16, "B16x64K"), (inputs.varlen_seqlens(32), 16, "config4"),
                              ([65536] * 16, 128, "H128")):
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        m.measure(seqlens, heads, label, iters=20)
    d = json.loads(buf.getvalue().strip().splitlines()[-1])
    print(f"PDL={os.environ['ETAP_PDL']} {label:10s} stream {d['us_per_step_stream']:8.2f} graph1 {d['us_per_step_graph']:8.2f} graph20 {d['us_per_step_graph20']:8.2f}", flush=True)
PY
done
