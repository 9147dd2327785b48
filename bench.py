# SPDX-License-Identifier: Apache-2.0
"""ETAP MLA decode benchmark (BASELINE.json metric) — prints ONE JSON line on rank 0.

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...      (N > 1)

Workload (BASELINE.json configs[1]): MLA decode, B=16 sequences x 64K latent-KV rows,
16 heads per GPU, d_qk=576 / d_v=512, bf16 paged KV (64-row pages), fp32 O + LSE.
A step = K2 (transposed tcgen05 pipeline; it computes the K1 split-KV schedule in its
prologue) + K3 (LSE combine) on inputs resident in HBM; with N > 1 GPUs every rank owns 16 of the 16*N heads (KV replicated)
and the step ends with the all-gather of O, fused into K2/K3 stores over NVLink peer memory (NCCL
all-gather when peer access is missing); weak scaling, SURVEY.md §8e. `e2e` is the same step with
host buffers: the C-ABI etap_mla_host_decode at N=1, the Python API on every rank at N > 1.
Inputs (1.2 GB of KV) exceed the 126 MB L2, so no flush is needed between steps.
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


def ncu_traffic() -> float | None:
    """DRAM read+write bytes per K2 launch at this workload from the committed ncu capture."""
    f = ROOT / "profiles" / "ncu_summary.json"
    if not f.exists():
        return None
    try:
        d = json.loads(f.read_text())
        return float(d["decode_kernel"]["dram_bytes_per_launch"]) if d.get("workload") == WORKLOAD else None
    except Exception:
        return None


def cpu_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def reference_cpu_sample(q_bits, kv_rows_bits, scale: float, nthreads: int):
    """Time the reference's run_etap (oracle/_ref, the unmodified etaplab library) on the
    given sample; returns seconds."""
    import numpy as np

    import oracle

    q = oracle.bf16_widen(q_bits)            # [B, H, 576]
    kv = oracle.bf16_widen(kv_rows_bits)     # [B, rows, 576]
    t, _, _ = oracle.ref_mla_run_etap_batch(np.ascontiguousarray(q), np.ascontiguousarray(kv), scale, nthreads)
    return t


def sample_inputs_cpu(inp, rows: int):
    """Contiguous first `rows` latent rows of every sequence as bf16 bits [B, rows, 576]."""
    import numpy as np
    import torch

    B = inp.batch
    pages = rows // 64
    idx = inp.block_table[:, :pages].long()                       # [B, pages]
    kv = inp.kv_pool[idx].reshape(B, pages * 64, 576)             # gather on device
    qb = inp.q[:, 0].contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    kvb = kv.contiguous().view(torch.int16).cpu().numpy().view(np.uint16)
    return qb, kvb


# ------------------------------------------------------------------------ reference arm
def run_reference(args) -> None:
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return  # rank 0 alone runs the CPU reference
    import numpy as np

    import oracle

    if not oracle.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libetaplab_ref.so not built"}))
        return
    rows = args.ref_rows
    threads = cpu_threads()
    # the same bf16 inputs as the GPU arm, generated on the host with the reference generator
    seeds = [42 + 7919 * b for b in range(BATCH)]
    q = np.stack([oracle.bf16_bits(oracle.ref_matrix_from_seed(HEADS, 576, 3 * s + 1)) for s in seeds])
    kv = np.stack([oracle.bf16_bits(oracle.ref_matrix_from_seed(rows, 576, 3 * s + 2)) for s in seeds])
    scale = 1.0 / math.sqrt(576.0)
    times = []
    for i in range(args.warmup + args.steps):
        t = reference_cpu_sample(q, kv, scale, threads)
        if i >= args.warmup:
            times.append(t)
    scale_up = CTX / rows
    us = float(np.median(times)) * 1e6 * scale_up
    sample = (f"run_etap exact64 (reference etaplab, compiled from source) on all {BATCH} sequences x "
              f"{rows} of {CTX} KV rows x {HEADS} heads per step, {threads} host threads (one per "
              f"sequence), median of {args.steps} steps scaled x{scale_up:.0f} to the full workload")
    line = {"metric": METRIC, "value": us, "unit": "us/step", "impl": "reference", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": us / 1e3, "higher_is_better": False,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch": BATCH, "ctx": CTX, "heads_per_gpu": HEADS,
                       "d_qk": 576, "d_v": 512},
            "cpu_baseline": {"value": us, "unit": "us/step", "cores": threads, "kind": "reference", "sample": sample},
            "e2e": {"value": us, "unit": "us/step", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------------ our arm
def run_ours(args) -> None:
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2506_01969_b200 import inputs, mla, sharding

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

    total_heads = HEADS * world
    seqlens = [CTX] * BATCH
    h0, _ = sharding.head_shard(total_heads, world, rank)
    inp = inputs.make_mla_inputs(seqlens, heads=HEADS, seed=42, device=dev, pad_value=0.0,
                                 head_offset=h0, total_heads=total_heads)
    plan = mla.MlaDecodePlan.create(BATCH, HEADS, dev)
    out = torch.empty((BATCH, 1, HEADS, 512), dtype=torch.float32, device=dev)
    lse = torch.empty((BATCH, 1, HEADS), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream(dev)
    # N > 1: the all-gather of O is fused into the kernels over NVLink peer memory
    # (etap_mla_decode_peer) when every local GPU pair has peer access; ETAP_GATHER=nccl (or no
    # peer access) uses decode + ncclAllGather instead
    gather = None
    if world > 1:
        gather = os.environ.get("ETAP_GATHER", "peer")
        ndev = torch.cuda.device_count()
        if gather == "peer" and not all(torch.cuda.can_device_access_peer(gpu, d) for d in range(ndev) if d != gpu):
            log("[bench] no peer access between all GPUs: falling back to NCCL all-gather")
            gather = "nccl"
        if gather == "peer":
            from paper_2506_01969_b200 import peer

            # every rank must take the same path: if the IPC setup fails anywhere (or the
            # first fused step does not verify against the NCCL gather), all fall back to NCCL
            ok = 1
            try:
                pg = peer.PeerGather(BATCH, HEADS, world, rank, device=dev)
            except Exception as e:  # noqa: BLE001
                log(f"[bench] rank {rank}: peer gather setup failed ({e})")
                pg, ok = None, 0
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
            if int(flag.item()) != 1:
                if pg is not None:
                    pg.close()
                gather = "nccl"

    # opt-in early metadata read (etap_mla.h ETAP_FLAG_EARLY_METADATA): nothing in this loop
    # writes seqlens / block_table, so K2 may read them before its grid dependency resolves
    dflags = mla.FLAG_EARLY_METADATA

    def step():
        # K2 computes the split schedule in its prologue (same partition as K1, which is the
        # per-step metadata call of the API and is off the critical path here) + K3 combine
        if gather == "peer":  # K2 + K3 store every rank's copy, K4 = arrival flags
            return pg.decode(plan, inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, flags=dflags)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse, flags=dflags)
        if world > 1:  # head-sharded output -> all 16*N heads on every rank (NCCL all-gather)
            return sharding.gather_heads(out), sharding.gather_heads(lse)
        return out, lse

    def barrier():
        if world > 1:
            if backend == "nccl":
                dist.barrier(device_ids=[local])
            else:
                dist.barrier()
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        for _ in range(args.steps):
            step()
        ev1.record(stream)
        torch.cuda.synchronize(dev)
    barrier()
    ms = ev0.elapsed_time(ev1) / args.steps
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    us = ms * 1e3

    # roofline pass: the dominant kernel (K2) timed alone with events on its stream
    k2_ms = []
    evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    for a, b in evs:
        a.record(stream)
        plan.decode(inp.q, inp.kv_pool, inp.block_table, inp.seqlens, inp.scale, out=out, lse=lse,
                    flags=mla.FLAG_SKIP_COMBINE)
        b.record(stream)
        plan.combine(out, lse)
    torch.cuda.synchronize(dev)
    k2_ms = sorted(a.elapsed_time(b) for a, b in evs)
    k2_avg_ms = sum(k2_ms) / len(k2_ms)

    nbytes = inputs.algorithmic_bytes(seqlens, HEADS)
    nflops = inputs.flops(seqlens, HEADS)
    peak, peak_kind = peaks()
    achieved = nbytes / (k2_avg_ms * 1e-3) / 1e9
    traffic = ncu_traffic()

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
        if world == 1 and args.e2e_steps > 0:
            e2e = e2e_host(inp, args.e2e_steps, dev)
            # serving-style step (cache resident in HBM): reported beside e2e, not instead
            e2e_serving = e2e_serving_host(inp, 50, dev)
        cpu = None
        if world == 1 and not args.no_cpu_baseline:
            cpu = cpu_baseline(inp, args)
        result = {
            "metric": METRIC, "value": us, "unit": "us/step", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": False, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": WORKLOAD, "batch": BATCH, "ctx": CTX, "heads_per_gpu": HEADS,
                       "total_heads": total_heads, "dist_backend": backend if world > 1 else None, "d_qk": 576, "d_v": 512, "page_rows": 64,
                       "kv_bytes_per_gpu": inp.kv_bytes(), "l2": "inputs (1.2 GB KV) > 126 MB L2, no flush",
                       "parallelism": (f"head-shard tp{world} (KV replicated, all-gather of O fused into K2/K3 "
                                       "over NVLink peer memory)" if gather == "peer" else
                                       f"head-shard tp{world} (KV replicated, NCCL all-gather of O)") if world > 1
                       else "single GPU", "decode_flags": "ETAP_FLAG_EARLY_METADATA (seqlens / block_table read "
                       "before the grid dependency; opt-in, nothing in the step writes them)",
                       "step": "K2 decode (in-kernel split schedule) + K3 combine" +
                       ((" + K4 peer arrival" if gather == "peer" else " + NCCL all-gather(O)") if world > 1 else "")},
            "throughput": {"hbm_gbs_aggregate": nbytes * world / (us * 1e-6) / 1e9,
                           "hbm_gbs_per_gpu": nbytes / (us * 1e-6) / 1e9,
                           "tflops_aggregate": nflops * world / (us * 1e-6) / 1e12,
                           "algorithmic_bytes_per_step_per_gpu": nbytes},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "kernel": "etap_mla_decode_kernel (K2)",
                         "kernel_avg_us": k2_avg_ms * 1e3, "peak_kind": peak_kind,
                         "timing": f"second timed pass of {args.steps} steps, CUDA events around each K2 launch"},
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


def cpu_baseline(inp, args) -> dict | None:
    try:
        import oracle

        if not oracle.ref_available():
            return None
        rows = args.cpu_rows
        threads = cpu_threads()
        qb, kvb = sample_inputs_cpu(inp, rows)
        t = reference_cpu_sample(qb, kvb, inp.scale, threads)
        scale_up = CTX / rows
        us = t * 1e6 * scale_up
        return {"value": us, "unit": "us/step", "cores": threads, "kind": "reference",
                "sample": (f"reference run_etap exact64 (oracle/_ref, etaplab compiled from source) on the same "
                           f"bf16 inputs: {BATCH} sequences x first {rows} of {CTX} rows x {HEADS} heads, "
                           f"{threads} threads, {t:.2f} s wall, scaled x{scale_up:.0f}")}
    except Exception as e:  # pragma: no cover
        log(f"[bench] cpu baseline failed: {e}")
        return None


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--cpu-rows", type=int, default=16384, help="KV rows per sequence in the CPU baseline sample")
    ap.add_argument("--ref-rows", type=int, default=2048, help="KV rows per sequence per reference-arm step")
    ap.add_argument("--no-cpu-baseline", action="store_true")
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
