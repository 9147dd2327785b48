# SPDX-License-Identifier: Apache-2.0
"""ETAP MLA decode benchmark (BASELINE.json metric) — prints ONE JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference] [--scaling strong]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Workload (BASELINE.json configs[1]): MLA decode, B=16 sequences x 64K latent-KV rows,
16 heads per GPU, d_qk=576 / d_v=512, bf16 paged KV (64-row pages), fp32 O + LSE.
A step = K2 (transposed tcgen05 pipeline; it computes the K1 split-KV schedule in its
prologue) + K3 (LSE combine) on inputs resident in HBM. Scaling (SURVEY.md §8e, configs[4]):
  * weak (default): every rank owns 16 heads, 16*N heads in total (KV replicated);
  * strong (--scaling strong --total-heads 128): the 128-head DeepSeek-R1 decode split over N
    ranks, 128/N heads each (N = 1: all 128 heads on one GPU).
With N > 1 the step ends with the all-gather of O, fused into K2/K3 stores over NVLink peer
memory (NCCL all-gather when peer access is missing). `e2e` is the same step with host
buffers: the C-ABI etap_mla_host_decode at N=1, the Python API on every rank at N > 1.
Inputs (1.2 GB of KV) exceed the 126 MB L2, so no flush is needed between steps.
`--impl reference` times the reference's own run_etap (exact64, oracle/_ref compiled from the
reference sources) on the full workload on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = json.loads((ROOT / "BASELINE.json").read_text())["metric"] if (ROOT / "BASELINE.json").exists() else \
    "MLA decode µs/step & HBM GB/s (B=16, ctx 64K, 16 heads/GPU); RMSE vs CPU"
BATCH, CTX, HEADS = 16, 65536, 16
WORKLOAD = "mla_decode_b16_ctx64k_h16_per_gpu"
SEED = 42


def workload(scaling: str, total_heads: int, world: int) -> tuple[str, int, int]:
    """(workload name, heads per rank, total heads) of a run."""
    if scaling == "strong":
        if total_heads % world or (total_heads // world) % 16:
            raise SystemExit(f"--total-heads {total_heads} cannot be split into {world} shards of 16k heads")
        return f"mla_decode_b16_ctx64k_h{total_heads}_strong", total_heads // world, total_heads
    return WORKLOAD, HEADS, HEADS * world


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------------ clocks (NVML)
class ClockSampler:
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x10: "sync_boost", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int, period_s: float = 0.002):
        self.samples, self.reasons, self.max_mhz = [], 0, None
        self.period, self.ok = period_s, False
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover - NVML missing
            log(f"[bench] NVML unavailable: {e}")
        self._stop = threading.Event()
        self._t = None

    def _run(self):
        while not self._stop.is_set():
            self.sample()
            time.sleep(self.period)

    def sample(self):
        if not self.ok:
            return
        try:
            self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
            self.reasons |= self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:
            pass

    def __enter__(self):
        self.sample()
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join()
        self.sample()

    def summary(self) -> dict:
        s = sorted(self.samples)
        med = s[len(s) // 2] if s else None
        names = [n for bit, n in self.REASONS.items() if self.reasons & bit and n != "gpu_idle"]
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": names, "samples": len(s)}


# ------------------------------------------------------------------------ helpers
def peaks() -> tuple[float, str]:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            return float(json.loads(p.read_text())["hbm_gbs"]), "measured"
        except Exception:
            pass
    return 6650.0, "fallback"


def ncu_traffic(name: str = WORKLOAD, world: int = 1) -> float | None:
    """DRAM read+write bytes per K2 launch at this workload from the committed ncu capture
    (profiles/ncu_summary.json: the headline K2, plus the FP8 and the 128-head single-GPU K2
    under "others", which match only the one-GPU run of those workloads)."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    try:
        d = json.loads(f.read_text())
        if name == WORKLOAD and d.get("workload") == WORKLOAD:
            return float(d["decode_kernel"]["dram_bytes_per_launch"])
        o = d.get("others", {}).get(name)
        return float(o["decode_kernel"]["dram_bytes_per_launch"]) if o and world == 1 else None
    except Exception:
        return None


def tensor_peak() -> tuple[float, str]:
    """Dense bf16 TF/s: the measured cuBLAS figure (MEASURED_PEAKS.json; sustained for a kernel
    inside a long step), else the B200_PROFILING fallback."""
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        try:
            d = json.loads(p.read_text())
            return float(d.get("bf16_tflops_sustained") or d["bf16_tflops"]), "measured (sustained)"
        except Exception:
            pass
    return 2250.0, "fallback (nominal dense bf16)"


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_full_step(heads: int, ctx: int, steps: int, warmup: int, threads: int) -> tuple[list[float], float]:
    """The reference's run_etap (exact64, oracle/_ref = the unmodified etaplab library compiled
    from source) on the FULL workload: B=16 problems of ctx rows x `heads` heads, generated once
    outside the timed region with the reference generator (the same bf16 operands the GPU arm
    reads), then `steps` timed steps (each all 16 problems, `threads` workers, like cmd_bench's
    timed loop over its problems, cli.cpp:277-283). Returns (step seconds, generation seconds)."""
    import oracle

    t0 = time.perf_counter()
    rb = oracle.RefMlaBench(BATCH, heads, ctx, SEED, 1.0 / math.sqrt(576.0), threads)
    gen = time.perf_counter() - t0
    try:
        times = []
        for i in range(warmup + steps):
            t = rb.step()
            if i >= warmup:
                times.append(t)
    finally:
        rb.close()
    return times, gen


# ------------------------------------------------------------------------ reference arm
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    import numpy as np

    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libetaplab_ref.so not built"}))
        return
    name, heads, total = workload(args.scaling, args.total_heads, world)
    ctx = args.ref_ctx
    threads = cpu_threads()
    times, gen = reference_full_step(heads, ctx, args.steps, args.warmup, threads)
    scale_up = CTX / ctx
    us = float(np.median(times)) * 1e6 * scale_up
    sample = (f"run_etap exact64 (reference etaplab, compiled from source by oracle/Makefile) on all {BATCH} "
              f"sequences x {ctx} KV rows x {heads} heads per step (TileConfig 64/64/2, bf16-rounded operands "
              f"from the reference generator, V = KV[:, :512]; {gen:.1f} s generation outside the timed region), "
              f"{threads} host threads over the batch, median of {args.steps} steps after {args.warmup} warm-up"
              + (f", scaled x{scale_up:g} from a reduced context" if ctx != CTX else " (full workload, not scaled)"))
    line = {"metric": METRIC, "value": us, "unit": "us/step", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": name, "batch": BATCH, "ctx": CTX, "heads_per_gpu": heads, "total_heads": total,
                       "d_qk": 576, "d_v": 512, "sample_ctx": ctx},
            "cpu_baseline": {"value": us, "unit": "us/step", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "step_times_s": times}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ our arm
def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_01969_b200 import _lib, inputs, mla, sharding

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        log(f"[bench] WORLD_SIZE={world} differs from --gpus {args.gpus}; using WORLD_SIZE")
    # ETAP_DIST_BACKEND=gloo lets the N>1 path run with several ranks on one GPU (testing only;
    # the driver's multi-GPU runs use NCCL, one rank per GPU)
    backend = os.environ.get("ETAP_DIST_BACKEND", "nccl")
    gpu = local % max(1, torch.cuda.device_count())
    torch.cuda.set_device(gpu)
    dev = torch.device("cuda", gpu)
    local = gpu
    if world > 1:
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    name, heads, total_heads = workload(args.scaling, args.total_heads, world)
    fp8 = args.kv == "fp8"
    if fp8:
        if world > 1:
            raise SystemExit("--kv fp8 runs on one GPU (the fused peer gather is bf16-only)")
        name += "_fp8kv"
    seqlens = [CTX] * BATCH
    h0, _ = sharding.head_shard(total_heads, world, rank)
    inp = inputs.make_mla_inputs(seqlens, heads=heads, seed=SEED, device=dev, pad_value=0.0,
                                 head_offset=h0, total_heads=total_heads)
    plan = mla.MlaDecodePlan.create(BATCH, heads, dev)
    out = torch.empty((BATCH, 1, heads, 512), dtype=torch.float32, device=dev)
    lse = torch.empty((BATCH, 1, heads), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    # N > 1: the all-gather of O is fused into the kernels over NVLink peer memory
    # (etap_mla_decode_peer) when every local GPU pair has peer access; ETAP_GATHER=nccl (or no
    # peer access) uses decode + ncclAllGather instead
    gather, fallback = None, None
    if world > 1:
        gather = os.environ.get("ETAP_GATHER", "peer")
        if gather != "peer":
            fallback = f"ETAP_GATHER={gather}"
        if gather == "peer":
            from paper_2506_01969_b200 import peer

            # every rank must take the same path: if the IPC setup fails anywhere (or the
            # first fused step does not verify against the NCCL gather), all fall back to NCCL
            ok = 1
            try:
                pg = peer.PeerGather(BATCH, heads, world, rank, device=dev)
            except Exception as e:  # noqa: BLE001  (peer.PeerAccessUnavailable: no P2P between some pair)
                log(f"[bench] rank {rank}: peer gather setup failed ({e}); falling back to the NCCL all-gather")
                pg, ok, fallback = None, 0, f"rank {rank}: {e}"
            fdev = dev if backend == "nccl" else "cpu"
            flag = torch.tensor([ok], device=fdev)
            dist.all_reduce(flag, op=dist.ReduceOp.MIN)
            if int(flag.item()) == 1:
                o_p, l_p = pg.decode(plan, inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale)
                plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse)
                o_n, l_n = sharding.gather_heads(out), sharding.gather_heads(lse)
                torch.cuda.synchronize(dev)
                same = int(torch.equal(o_p.reshape(o_n.shape), o_n) and torch.equal(l_p.reshape(l_n.shape), l_n))
                flag = torch.tensor([same], device=fdev)
                dist.all_reduce(flag, op=dist.ReduceOp.MIN)
                if int(flag.item()) != 1:
                    log("[bench] fused peer gather differs from the NCCL gather: falling back to NCCL")
                    fallback = "fused peer gather differs from the NCCL gather"
            if int(flag.item()) != 1:
                fallback = fallback or "peer gather setup failed on another rank"
                if pg is not None:
                    pg.close()
                gather = "nccl"

    # opt-in (etap_mla.h ETAP_FLAG_INDEPENDENT_INPUTS, implies ETAP_FLAG_EARLY_METADATA): the kernel
    # before each K2 in this loop is the previous step's K3, which writes only O / LSE, so K2
    # reads seqlens / block_table / Q / KV without waiting for it and waits only before its
    # first global write
    dflags = mla.FLAG_INDEPENDENT_INPUTS
    KV_SCALE = 0.125  # dequantised value = KV_SCALE * e4m3 (the scale the GPU tests and sweeps use)
    kv8 = (inp.kv_pool.float() / KV_SCALE).to(torch.float8_e4m3fn) if fp8 else None

    def step():
        if fp8:  # K2-FP8 (kind::f8f6f4 UMMAs straight from the fp8 pages) + K3
            plan.decode_fp8(inp.q, kv8, inp.block_table, inp.seqlens, inp.scale, KV_SCALE, out=out, lse=lse,
                            flags=dflags)
            return out, lse
        # K2 computes the split schedule in its prologue (same partition as K1, which is the
        # per-step metadata call of the API and is off the critical path here) + K3 combine
        if gather == "peer":  # K2 + K3 store every rank's copy, K4 = arrival flags
            return pg.decode(plan, inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=dflags)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse, flags=dflags)
        if world > 1:  # head-sharded output -> all heads on every rank (NCCL all-gather)
            return sharding.gather_heads(out), sharding.gather_heads(lse)
        return out, lse

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize(dev)

    # K2's span per launch without touching programmatic launch (events around K2 would
    # serialise it): the product kernel stamps %globaltimer per CTA when its grid dependency
    # resolved and at exit (etap_mla_debug_span); one row of stamps per timed step
    L = _lib.lib()
    spans = torch.zeros((args.steps, plan.num_sm_parts, 2), dtype=torch.int64, device=dev)
    for _ in range(args.warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for i in range(args.steps):
            L.etap_mla_debug_span(spans[i].data_ptr())
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    L.etap_mla_debug_span(None)
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    # The same K steps without the overlap of consecutive steps (ETAP_FLAG_EARLY_METADATA only:
    # every decode waits for the previous step's combine before its loads), reported beside
    ms_dep = None
    if world == 1 and gather is None:
        dflags_run = dflags
        dflags = mla.FLAG_EARLY_METADATA
        for _ in range(3):
            step()
        torch.cuda.synchronize(dev)
        ev0.record(stream)
        for i in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
        ms_dep = ev0.elapsed_time(ev1) / args.steps
        dflags = dflags_run
    # Same-box read-only streaming bound over the same paged pool (after the timed region, not
    # part of any step): the TMA stream kernel (etap_mla_stream_bench) reads every page once with
    # no compute. MEASURED_PEAKS.json's figure is a read+write copy, which a read-only stream
    # exceeds, so roofline.frac against it can pass 1; read_stream.frac is the tighter ratio.
    read_stream = None
    if world == 1:
        pages_all = int(inp.kv_pool.shape[0])
        rs = []
        for grid, nslot in ((296, 24), (148, 24)):
            ppc = pages_all // grid
            for _ in range(3):
                _lib.check(L.etap_mla_stream_bench(inp.kv_pool.data_ptr(), pages_all, ppc, grid, nslot, stream.cuda_stream),
                           "etap_mla_stream_bench")
            ev0.record(stream)
            for _ in range(20):
                L.etap_mla_stream_bench(inp.kv_pool.data_ptr(), pages_all, ppc, grid, nslot, stream.cuda_stream)
            ev1.record(stream)
            torch.cuda.synchronize(dev)
            rs.append(ppc * grid * inputs.PAGE_ROWS * 576 * 2 / (ev0.elapsed_time(ev1) / 20 * 1e-3) / 1e9)
        read_stream = max(rs)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    us = ms * 1e3
    sp = spans.cpu().numpy()
    # Per launch: the mean over CTAs of each CTA's busy span (first KV load -> exit). With
    # ETAP_FLAG_INDEPENDENT_INPUTS consecutive launches overlap (the next step's CTAs start on SMs
    # this step's CTAs leave, during its tail), so first-start -> last-exit of one launch is not
    # its duration; every CTA streams its 1/148 share of the bytes within its own span.
    # A launch's duration: first CTA start -> last CTA exit, but counting time it overlaps the
    # previous launch only once, i.e. min(that span, last exit - the previous launch's last
    # exit). Without the step overlap this is the launch span; with it, the exit-to-exit period
    # of consecutive launches. (The mean CTA busy span undercounts: L2 prefetches issued before
    # a CTA's first stamp and the next step's early start move bytes outside the spans; the
    # slowest CTA's span overcounts: it includes the time it ran beside the previous launch.)
    cta_us = (sp[:, :, 1] - sp[:, :, 0]) / 1e3
    first, last = sp[:, :, 0].min(axis=1), sp[:, :, 1].max(axis=1)
    k2_us = (last - first) / 1e3
    k2_us[1:] = np.minimum(k2_us[1:], (last[1:] - last[:-1]) / 1e3)
    k2_avg_us = float(k2_us.mean())
    k2_mean_cta_us = float(cta_us.mean())
    launch_span_us = float(((sp[:, :, 1].max(axis=1) - sp[:, :, 0].min(axis=1)) / 1e3).mean())

    unit_heads, _parts = mla.schedule_unit(heads, plan.num_sm_parts)
    pair = unit_heads == 128
    nbytes = inputs.algorithmic_bytes(seqlens, heads)
    if fp8:  # the latent cache is one byte per element
        nbytes -= sum(seqlens) * 576
    nflops = inputs.flops(seqlens, heads)
    peak, peak_kind = peaks()
    tpeak, tpeak_kind = tensor_peak()
    achieved = nbytes / (k2_avg_us * 1e-6) / 1e9
    achieved_tf = nflops / (k2_avg_us * 1e-6) / 1e12
    # arithmetic intensity vs the ridge: 16 heads (30 FLOP/B) are HBM-bound, 128 heads (242) sit
    # at the ridge (peak TF/s / peak GB/s ~ 251)
    bound = "hbm" if nflops / nbytes < tpeak * 1e12 / (peak * 1e9) else "tensor"
    traffic = ncu_traffic(name, world)

    # N > 1 e2e: every rank, through the Python API, with host buffers (all ranks take part)
    e2e_multi = None
    if world > 1 and args.e2e_steps > 0:
        def run_step(q, kv, bt, sl):
            if gather == "peer":
                return pg.decode(plan, q, kv, bt, sl, inp.scale)
            plan.decode(q, kv, bt, sl, inp.scale, out=out, lse=lse)
            return sharding.gather_heads(out), sharding.gather_heads(lse)
        e2e_multi = e2e_ranks(inp, args.e2e_steps, dev, run_step, barrier, world)

    result = {}
    if rank == 0:
        clocks = clk.summary()
        # e2e: the reference-facing C-ABI call with HOST buffers (H2D + K1/K2/K3 + D2H per step)
        e2e, e2e_serving = e2e_multi, None
        if world == 1 and args.e2e_steps > 0 and fp8:
            e2e = e2e_fp8(inp, kv8, KV_SCALE, plan, args.e2e_steps, dev)
        elif world == 1 and args.e2e_steps > 0:
            e2e = e2e_host(inp, args.e2e_steps, dev)
            # serving-style step (cache resident in HBM): reported beside e2e, not instead
            e2e_serving = None if fp8 else e2e_serving_host(inp, 50, dev)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(heads, args)
        if bound == "hbm":
            roof = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                    "peak_kind": peak_kind, "tensor_frac": achieved_tf / tpeak}
        else:
            roof = {"bound": "tensor", "achieved": achieved_tf, "peak": tpeak, "unit": "TFLOP/s",
                    "frac": achieved_tf / tpeak, "peak_kind": tpeak_kind, "hbm_frac": achieved / peak,
                    "note": "useful FLOPs 2*H*ctx*(576+512); the bf16 hi+lo split of P doubles the issued GEMM2 "
                            "FLOPs (1.47x useful) and is not credited"}
        kname = ("etap_mla_decode_fp8_kernel (K2-FP8)" if fp8 else
                 "etap_mla_decode_pair_kernel (K2, CTA pairs)" if pair else "etap_mla_decode_kernel (K2)")
        if read_stream is not None:
            roof["read_stream"] = {
                "gbs": read_stream, "frac": achieved / read_stream, "step_frac": nbytes / (us * 1e-6) / 1e9 / read_stream,
                "how": "etap_mla_stream_bench: TMA page stream over this run's pool, no compute, best of grid 296/148 "
                       "x 24 slots, 20 launches, CUDA events; step_frac = algorithmic bytes / whole step time"}
        roof.update({"traffic": traffic, "kernel": kname, "kernel_avg_us": k2_avg_us,
                     "kernel_min_us": float(k2_us.min()), "kernel_max_us": float(k2_us.max()),
                     "kernel_mean_cta_span_us": k2_mean_cta_us,
                     "launch_span_us": launch_span_us,
                     "timing": (f"%globaltimer stamps of the product K2 over the {args.steps} timed steps "
                                "(etap_mla_debug_span: per CTA, first KV load and exit), programmatic launch "
                                "intact; kernel_avg_us = mean over launches of min(first CTA start -> last CTA exit, last exit - "
                                "the previous launch's last exit): consecutive launches overlap, and the overlap "
                                "is counted once; launch_span_us = first start -> last exit, overlap included)")})
        result = {
            "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "e4m3 latent cache, fp32 accumulate" if fp8 else "bf16",
            "data": "synthetic",
            "config": {"workload": name, "batch": BATCH, "ctx": CTX, "heads_per_gpu": heads,
                       "total_heads": total_heads, "dist_backend": backend if world > 1 else None, "d_qk": 576,
                       "d_v": 512, "page_rows": 64, "head_group": unit_heads,
                       "work_unit": (f"{unit_heads} heads on a CTA pair (tcgen05 cta_group::2)" if pair
                                     else f"{unit_heads} heads on one CTA"),
                       "kv_bytes_per_gpu": inp.kv_bytes(), "l2": "inputs (1.2 GB KV) > 126 MB L2, no flush",
                       "parallelism": (f"head-shard tp{world} (KV replicated, all-gather of O fused into K2/K3 "
                                       "over NVLink peer memory)" if gather == "peer" else
                                       f"head-shard tp{world} (KV replicated, NCCL all-gather of O)") if world > 1
                       else "single GPU", "gather_fallback_reason": fallback, "decode_flags": "ETAP_FLAG_INDEPENDENT_INPUTS (opt-in, implies ETAP_FLAG_EARLY_METADATA: "
                       "the kernel before each decode is the previous step's combine, which writes none of the "
                       "decode's inputs, so the decode loads KV / Q / seqlens / block_table without waiting for "
                       "it and waits for it only before its first global write)",
                       "us_per_step_without_step_overlap": (ms_dep * 1e3 if ms_dep is not None else None),
                       "step": "K2 decode (in-kernel split schedule) + K3 combine" +
                       ((" + K4 peer arrival" if gather == "peer" else " + NCCL all-gather(O)") if world > 1 else "")},
            "throughput": {"hbm_gbs_aggregate": nbytes * world / (us * 1e-6) / 1e9,
                           "hbm_gbs_per_gpu": nbytes / (us * 1e-6) / 1e9,
                           "tflops_aggregate": nflops * world / (us * 1e-6) / 1e12,
                           "tflops_per_gpu": nflops / (us * 1e-6) / 1e12,
                           "algorithmic_bytes_per_step_per_gpu": nbytes, "flops_per_step_per_gpu": nflops},
            "roofline": roof,
            "clocks": clocks,
            "gpu_launches": (3 if gather == "peer" else 2) * args.steps,
            "e2e": e2e,
            "e2e_serving": e2e_serving,
            "cpu_baseline": cpu,
        }
        print(json.dumps(result), flush=True)
    if world > 1:
        barrier()
        if gather == "peer":
            pg.close()
        dist.destroy_process_group()


def e2e_host(inp, steps: int, dev) -> dict:
    """Same workload through etap_mla_host_decode (pinned host buffers in, host results out)."""
    import ctypes as C

    import torch

    from paper_2506_01969_b200 import _lib

    L = _lib.lib()
    q = inp.q.cpu().pin_memory()
    kv = inp.kv_pool.cpu().pin_memory()
    bt = inp.block_table.cpu().pin_memory()
    sl = inp.seqlens.cpu().pin_memory()
    out = torch.empty((inp.batch, inp.heads, 512), dtype=torch.float32).pin_memory()
    lse = torch.empty((inp.batch, inp.heads), dtype=torch.float32).pin_memory()
    ctx = C.c_void_p()
    _lib.check(L.etap_mla_host_ctx_create(inp.batch, inp.heads, kv.shape[0], bt.shape[1], C.byref(ctx)), "ctx")
    try:
        def call():
            _lib.check(L.etap_mla_host_decode(ctx, q.data_ptr(), kv.data_ptr(), bt.data_ptr(), sl.data_ptr(),
                                              inp.scale, 0, out.data_ptr(), lse.data_ptr()), "host_decode")
        call()
        t0 = time.perf_counter()
        for _ in range(steps):
            call()
        dt = (time.perf_counter() - t0) / steps
    finally:
        L.etap_mla_host_ctx_destroy(ctx)
    h2d = q.numel() * 2 + kv.numel() * 2 + bt.numel() * 4 + sl.numel() * 4
    d2h = out.numel() * 4 + lse.numel() * 4
    # the bound of this path: a plain pinned host->device copy of the same bytes
    dst = torch.empty_like(kv, device=dev)
    dst.copy_(kv, non_blocking=True)
    torch.cuda.synchronize(dev)
    t0 = time.perf_counter()
    for _ in range(2):
        dst.copy_(kv, non_blocking=True)
    torch.cuda.synchronize(dev)
    h2d_gbs = 2 * kv.numel() * 2 / (time.perf_counter() - t0) / 1e9
    del dst
    return {"value": dt * 1e6, "unit": "us/step", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "etap_mla_host_decode (C-ABI, pinned host buffers, synchronous)", "steps": steps,
            "bound": {"kind": "pcie_h2d", "measured_h2d_gbs": h2d_gbs,
                      "bound_us": (h2d + d2h) / h2d_gbs / 1e3, "frac": (h2d + d2h) / h2d_gbs / 1e3 / (dt * 1e6)}}


def e2e_fp8(inp, kv8, kv_scale: float, plan, steps: int, dev) -> dict:
    """FP8 cache, end to end through the Python API (decode_fp8 has no host-buffer C-ABI entry):
    per step the Q, the fp8 latent cache, the block table and seqlens are copied from pinned host
    memory, the step runs, O / LSE are read back into pinned host memory; wall clock."""
    import torch

    host = [t.cpu().pin_memory() for t in (inp.q, kv8, inp.block_table, inp.seqlens)]
    devb = [torch.empty_like(t) for t in (inp.q, kv8, inp.block_table, inp.seqlens)]
    out_h = torch.empty((inp.batch, 1, inp.heads, 512), dtype=torch.float32).pin_memory()
    lse_h = torch.empty((inp.batch, 1, inp.heads), dtype=torch.float32).pin_memory()

    def call():
        for d, h in zip(devb, host):
            d.copy_(h, non_blocking=True)
        o, l = plan.decode_fp8(devb[0], devb[1], devb[2], devb[3], inp.scale, kv_scale)
        out_h.copy_(o, non_blocking=True)
        lse_h.copy_(l, non_blocking=True)
        torch.cuda.synchronize(dev)

    call()
    t0 = time.perf_counter()
    for _ in range(steps):
        call()
    dt = (time.perf_counter() - t0) / steps
    h2d = sum(t.numel() * t.element_size() for t in host)
    d2h = out_h.numel() * 4 + lse_h.numel() * 4
    return {"value": dt * 1e6, "unit": "us/step", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "MlaDecodePlan.decode_fp8 (Python API over the C-ABI, pinned host buffers, synchronous)",
            "steps": steps}


def e2e_ranks(inp, steps: int, dev, run_step, barrier, world: int) -> dict:
    """N > 1: the same step end to end on every rank through the Python API (head-sharded
    decode + all-gather of O): per step each rank copies its Q shard, the replicated latent
    cache, the block table and seqlens from pinned host buffers, runs the step and reads the
    gathered O / LSE (all 16*N heads) back into pinned host memory. Wall clock per rank between
    barriers, max over ranks."""
    import torch
    import torch.distributed as dist

    host = [t.cpu().pin_memory() for t in (inp.q, inp.kv_pool, inp.block_table, inp.seqlens)]
    devb = [torch.empty_like(t) for t in (inp.q, inp.kv_pool, inp.block_table, inp.seqlens)]
    res_h = []

    def one():
        for d, h in zip(devb, host):
            d.copy_(h, non_blocking=True)
        o, l = run_step(*devb)
        if not res_h:
            res_h.extend([torch.empty(o.shape, dtype=o.dtype).pin_memory(), torch.empty(l.shape, dtype=l.dtype).pin_memory()])
        res_h[0].copy_(o, non_blocking=True)
        res_h[1].copy_(l, non_blocking=True)
        torch.cuda.synchronize(dev)

    one()
    barrier()
    t0 = time.perf_counter()
    for _ in range(steps):
        one()
    dt = (time.perf_counter() - t0) / steps
    t = torch.tensor([dt], device=dev if dist.get_backend() == "nccl" else "cpu", dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    h2d = sum(h.numel() * h.element_size() for h in host)
    d2h = sum(r.numel() * r.element_size() for r in res_h)
    del devb
    return {"value": float(t.item()) * 1e6, "unit": "us/step", "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps,
            "api": f"paper_2506_01969_b200 Python API on each of {world} ranks (pinned host buffers in: Q shard + "
                   "replicated latent cache + block table + seqlens; head-sharded decode + all-gather of O; "
                   "all heads' O / LSE out), wall clock, max over ranks"}


def e2e_serving_host(inp, steps: int, dev) -> dict:
    """A serving decode step through the C-ABI against a cache resident in HBM
    (etap_mla_host_ctx_load once, untimed; then etap_mla_host_decode_step per step): each step
    copies Q, one new latent row per sequence and seqlens host->device, appends the rows into
    the paged pool, decodes at the full context and copies O / LSE back. The appended row is
    the context's last row, so every step is the same 64K-context decode as `value`."""
    import ctypes as C

    import torch

    from paper_2506_01969_b200 import _lib

    L = _lib.lib()
    q = inp.q.cpu().pin_memory()
    bt_d = inp.block_table
    last = (inp.seqlens.long() - 1).clamp(min=0)
    pages = bt_d.gather(1, (last // 64).unsqueeze(1)).squeeze(1).long()
    rows = inp.kv_pool[pages, last % 64].contiguous().cpu().pin_memory()    # [B, 576] bf16
    sl = inp.seqlens.cpu().pin_memory()
    out = torch.empty((inp.batch, inp.heads, 512), dtype=torch.float32).pin_memory()
    lse = torch.empty((inp.batch, inp.heads), dtype=torch.float32).pin_memory()
    ctx = C.c_void_p()
    _lib.check(L.etap_mla_host_ctx_create(inp.batch, inp.heads, inp.kv_pool.shape[0], bt_d.shape[1], C.byref(ctx)),
               "ctx")
    try:
        kv_h = inp.kv_pool.cpu().pin_memory()
        bt_h = bt_d.cpu().pin_memory()
        _lib.check(L.etap_mla_host_ctx_load(ctx, kv_h.data_ptr(), bt_h.data_ptr()), "ctx_load")
        del kv_h

        def call():
            _lib.check(L.etap_mla_host_decode_step(ctx, q.data_ptr(), rows.data_ptr(), sl.data_ptr(), inp.scale, 0,
                                                   out.data_ptr(), lse.data_ptr()), "host_decode_step")
        for _ in range(3):
            call()
        t0 = time.perf_counter()
        for _ in range(steps):
            call()
        dt = (time.perf_counter() - t0) / steps
    finally:
        L.etap_mla_host_ctx_destroy(ctx)
    h2d = q.numel() * 2 + rows.numel() * 2 + sl.numel() * 4
    d2h = out.numel() * 4 + lse.numel() * 4
    return {"value": dt * 1e6, "unit": "us/step", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "api": "etap_mla_host_decode_step (C-ABI, cache resident in HBM; per step H2D of Q + one new latent "
                   "row per sequence + seqlens, append, decode, D2H of O/LSE, synchronous)", "steps": steps}


def cpu_baseline(heads: int, args) -> dict | None:
    """The reference's CPU path on this box's host cores: full steps (all 16 sequences x 64K
    rows) of run_etap exact64 after one warm-up step, on the same operands as the GPU arm; the
    median of 3 steps at 16 heads (one step above: 128 heads take ~4 s per step)."""
    try:
        import oracle

        if not oracle.ref_available():
            return None
        threads = cpu_threads()
        nsteps = 3 if heads <= 16 else 1
        times, gen = reference_full_step(heads, args.cpu_ctx, nsteps, 1, threads)
        scale_up = CTX / args.cpu_ctx
        med = sorted(times)[len(times) // 2]
        us = med * 1e6 * scale_up
        return {"value": us, "unit": "us/step", "cores": threads, "kind": "reference",
                "sample": (f"reference run_etap exact64 (oracle/_ref, etaplab compiled from source) on {BATCH} "
                           f"sequences x {args.cpu_ctx} rows x {heads} heads, the GPU arm's operands (reference "
                           f"generator, bf16-rounded, V = KV[:, :512]; {gen:.1f} s generation untimed), {threads} "
                           f"threads, median of {nsteps} step(s) after one warm-up step, {med:.2f} s wall"
                           + (f", scaled x{scale_up:g}" if args.cpu_ctx != CTX else " (full workload, not scaled)"))}
    except Exception as e:  # pragma: no cover
        log(f"[bench] cpu baseline failed: {e}")
        return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--scaling", choices=["weak", "strong"], default="weak",
                    help="weak: 16 heads per GPU (16*N total); strong: --total-heads split over N GPUs")
    ap.add_argument("--total-heads", type=int, default=128, help="heads of the strong-scaling workload")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-ctx", type=int, default=CTX, help="KV rows per sequence of the CPU baseline step")
    ap.add_argument("--ref-ctx", type=int, default=CTX, help="KV rows per sequence of each reference-arm step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--kv", choices=["bf16", "fp8"], default="bf16",
                    help="latent cache format: bf16 (the headline) or fp8 e4m3 (K2-FP8, single GPU)")
    args = ap.parse_args()
    if args.warmup < 3:
        log("[bench] warmup raised to 3 (contract minimum)")
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
