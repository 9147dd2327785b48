# SPDX-License-Identifier: Apache-2.0
"""Summarise an ncu capture of the decode kernel (K2) and a launch list into profiles/.

    python scripts/ncu_summary.py gpurun_out/prof_r01.ncu-rep gpurun_out/launches_r01.csv r01
writes profiles/ncu_summary.json (read by bench.py for roofline.traffic) and
profiles/<tag>/ncu_decode_kernel.md.
"""
from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "sm__cycles_elapsed.avg", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "lts__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed", "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "nsecond": 1e-9, "msecond": 1e-3,
         "us": 1e-6, "ns": 1e-9}


def raw(rep: str) -> dict:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in KEYS:
            try:
                d[h] = (float(v.replace(",", "")), u)
            except ValueError:
                d[h] = (v, u)
    return d


def main() -> None:
    fp8 = "--fp8" in sys.argv  # FP8 kernel capture: profiles/<tag>/ncu_fp8_kernel.md only
    heads = 16
    if "--heads" in sys.argv:  # other head counts: profiles/<tag>/ncu_decode_kernel_h<H>.md only
        heads = int(sys.argv[sys.argv.index("--heads") + 1])
    args = [a for i, a in enumerate(sys.argv[1:], 1) if a not in ("--fp8", "--heads") and sys.argv[i - 1] != "--heads"]
    rep, launches, tag = args[0], args[1] if len(args) > 1 and args[1] != "-" else None, args[2] if len(args) > 2 else "r01"
    from paper_2506_01969_b200 import inputs

    d = raw(rep)
    rd = d["dram__bytes_read.sum"][0] * SCALE[d["dram__bytes_read.sum"][1]]
    wr = d["dram__bytes_write.sum"][0] * SCALE[d["dram__bytes_write.sum"][1]]
    dur = d["gpu__time_duration.sum"][0] * SCALE[d["gpu__time_duration.sum"][1]]
    alg = inputs.algorithmic_bytes([65536] * 16, heads)
    flops = inputs.flops([65536] * 16, heads)
    if fp8:  # the latent cache is one byte per element
        alg -= 65536 * 16 * 576
    summary = {
        "workload": "mla_decode_b16_ctx64k_h16_per_gpu" if heads == 16 else f"mla_decode_b16_ctx64k_h{heads}",
        "tag": tag, "source": rep,
        "decode_kernel": {
            "dram_bytes_read": rd, "dram_bytes_write": wr, "dram_bytes_per_launch": rd + wr,
            "algorithmic_bytes": alg, "traffic_over_algorithmic": (rd + wr) / alg,
            "duration_us_cold_serialised": dur * 1e6,
            "dram_throughput_pct_of_ncu_peak": d["gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"][0],
            "tensor_pipe_active_pct": d["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"][0],
            "tc_issue_pipe_active_pct": d.get("sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_elapsed", (None,))[0],
            "useful_tflops_at_capture": flops / dur / 1e12,
            "sm_throughput_pct": d["sm__throughput.avg.pct_of_peak_sustained_elapsed"][0],
            "sm_clock_ghz": d["sm__cycles_elapsed.avg"][0] / dur / 1e9,
            "registers_per_thread": d["launch__registers_per_thread"][0],
            "grid": d["launch__grid_size"][0], "block": d["launch__block_size"][0],
            "l2_hit_rate_pct": d["lts__t_sector_hit_rate.pct"][0],
        },
    }
    if launches and Path(launches).exists():
        rows = [r for r in csv.DictReader(l for l in open(launches) if not l.startswith("==")) if r.get("Metric Name") == "gpu__time_duration.sum"]
        ks = {}
        for r in rows:
            name = r["Kernel Name"].replace("<unnamed>::", "").replace("void ", "").split("(")[0].split("<")[0]
            ks.setdefault(name, []).append(float(r["Metric Value"]) * SCALE.get(r["Metric Unit"], 1e-9))
        tot = sum(sum(v) for v in ks.values())
        summary["launch_list"] = {k: {"launches": len(v), "avg_us": sum(v) / len(v) * 1e6,
                                      "share": sum(v) / tot} for k, v in ks.items()}
    # profiles/ncu_summary.json: the headline K2 at top level (bench.py roofline.traffic), the
    # FP8 and other-head-count captures under "others", keyed by bench.py's config.workload
    f = ROOT / "profiles" / "ncu_summary.json"
    old = json.loads(f.read_text()) if f.exists() else {}
    others = old.get("others", {})
    if not fp8 and heads == 16:
        out = dict(summary, others=others)
    else:
        key = "mla_decode_b16_ctx64k_h16_per_gpu_fp8kv" if fp8 else f"mla_decode_b16_ctx64k_h{heads}_strong"
        others[key] = {"tag": tag, "source": rep, "decode_kernel": summary["decode_kernel"]}
        out = dict(old, others=others)
    f.write_text(json.dumps(out, indent=1) + "\n")
    tagdir = ROOT / "profiles" / tag
    tagdir.mkdir(parents=True, exist_ok=True)
    kname = ("etap_mla_decode_fp8_kernel (K2-FP8, e4m3 latent cache)" if fp8 else
             "etap_mla_decode_pair_kernel (K2, CTA pairs)" if heads % 128 == 0 else "etap_mla_decode_kernel (K2)")
    lines = [f"# ncu — {kname}, B=16 x 64K, {heads} heads ({tag})", "",
             f"source: `{rep}` (`ncu --set full --clock-control none --import-source on`, one launch)", "",
             "| metric | value |", "|---|---|"]
    for k, v in summary["decode_kernel"].items():
        lines.append(f"| {k} | {v:.6g} |" if isinstance(v, float) else f"| {k} | {v} |")
    if "launch_list" in summary:
        lines += ["", "## launch list (cold, serialised: compare shares)", "", "| kernel | launches | avg us | share |",
                  "|---|---|---|---|"]
        for k, v in summary["launch_list"].items():
            lines.append(f"| {k} | {v['launches']} | {v['avg_us']:.2f} | {v['share']:.3f} |")
    fname = "ncu_fp8_kernel.md" if fp8 else ("ncu_decode_kernel.md" if heads == 16 else f"ncu_decode_kernel_h{heads}.md")
    (tagdir / fname).write_text("\n".join(lines) + "\n")
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main()
