#!/usr/bin/env python
"""Benchmark of the HA-RAG hot path on B200 (BASELINE.json metric:
"assembled-KV GB/s & per-request assemble latency vs HBM/link roofline").

A step = one batch of B requests through the whole online path: a6 request
planning, a8 fused gather-dequantise-scatter (one kernel launch for the
HBM-resident set), a1 hotness counting fused in the kernel, and every
--epoch-every steps a9 (hotness all-reduce over NCCL when N > 1, decay,
re-rank, re-placement).  Compression (a2-a5) is build time ("compress once",
S:336; Alg. 1 is offline) and is reported separately under "build".

  python bench.py [--gpus N] [--steps K] [--warmup W] [--workload c2|tiny] [--impl ours|reference]

N > 1 runs under torchrun: KV heads are sharded across ranks (each rank
assembles its H/N heads of every request; strong scaling, no data-path
collective).  Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "assembled-KV GB/s & per-request assemble latency vs HBM/link roofline, 1/2/4/8 GPU"
PAPER_LADDER = ("INT8", "FP8E4M3", "FP8E5M2", "GSE8")
NORTH_LADDER = ("PASS16", "INT8", "INT4")

WORKLOADS = {
    # BASELINE.json configs[1]: Llama-3-8B KV shape, 512-token chunks, Zipf hotness, top-k 10.
    # HBM-resident sub-store of 2,000 docs; paper ladder and thresholds.
    "c2": dict(L=32, H=8, D=128, T=512, n_docs=2000, k=10, batch=32, s=1.1, dtype="bf16",
               ladder=PAPER_LADDER, taus=(0.1, 0.1, 0.1), desc="Llama-3-8B KV shape (32 layers x 8 KV heads x "
               "head_dim 128), 2,000-doc HBM-resident store of 512-token chunks, Zipf(1.1) hotness, top-k 10, "
               "batch 32 requests, paper ladder INT8/E4M3/E5M2/GSE-8 at 10/10/10/70%"),
    # BASELINE.json configs[0]
    "tiny": dict(L=2, H=2, D=64, T=64, n_docs=16, k=4, batch=8, s=1.1, dtype="fp16", ladder=NORTH_LADDER,
                 taus=(0.25, 0.25), desc="tiny store: 16 chunks x 64 tokens, 2 layers, 2 KV heads, head_dim 64, "
                 "fp16, PASS16/INT8/INT4 mix, top-k 4"),
}

BYTES_READ = {"PASS16": 2.0, "FP8E4M3": 1.0, "FP8E5M2": 1.0, "INT4": 0.5}


def env_int(k, d):
    return int(os.environ.get(k, d))


def clocks_sampler(device: int):
    """Sample nvidia-smi clocks and throttle reasons while the timed region runs."""
    q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", "-i", str(device), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                              "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except OSError:
        return None, None
    rows: list[list[str]] = []

    def reader():
        for line in p.stdout:
            rows.append([x.strip() for x in line.split(",")])

    t = threading.Thread(target=reader, daemon=True)
    t.start()
    return p, rows


def clocks_summary(p, rows):
    if p is None:
        return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
    time.sleep(0.15)
    p.terminate()
    try:
        p.wait(2)
    except subprocess.TimeoutExpired:
        p.kill()
    sm, mx, reasons = [], [], set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for r in rows:
        try:
            sm.append(float(r[0]))
            mx.append(float(r[1]))
        except (ValueError, IndexError):
            continue
        for n, v in zip(names, r[4:8]):
            if v.strip().lower() == "active":
                reasons.add(n)
    return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
            "reasons": sorted(reasons), "samples": len(sm)}


def alg_bytes_per_elem(scheme: str, G: int) -> float:
    if scheme == "INT8":
        return 1.0 + 4.0 / G + 2.0
    if scheme == "GSE8":
        return 1.0 + 16.0 / 65536 + 2.0
    if scheme == "INT4":
        return 0.5 + 8.0 / G + 2.0
    return BYTES_READ[scheme] + 2.0


# ------------------------------------------------------------------ oracle
class OracleSample:
    """The CPU oracle on a bounded sample of the workload: request 0 of the
    first batch, restricted to the first `layers` layers (all heads).  Packed
    blobs are prepared once (compression is offline); what is timed is the
    oracle's assemble = decode + scatter, the same work the GPU step does."""

    def __init__(self, wl, req, layers: int):
        from oracle import hotness
        from oracle import store as ost
        import synth
        L, H, D, T, k = wl["L"], wl["H"], wl["D"], wl["T"], wl["k"]
        self.ost, self.wl, self.layers = ost, wl, layers
        self.lay = ost.Layout(L=layers, H=H, T=T, D=D, dtype=wl["dtype"])
        prof = synth.gen_requests(wl["n_docs"], 4 * wl["n_docs"], k, wl["s"], seed=7)
        h = hotness.count_requests(prof, wl["n_docs"]).astype(np.uint64)
        names = {"PASS16": ost.PASS16, "INT8": ost.INT8, "FP8E4M3": ost.FP8E4M3, "FP8E5M2": ost.FP8E5M2,
                 "GSE8": ost.GSE8, "INT4": ost.INT4}
        self.schemes = hotness.assign_schemes(h.tolist(), [names[s] for s in wl["ladder"]], wl["taus"])
        self.req = [int(d) for d in req]
        self.blobs = {}
        for d in self.req:
            for kind in (0, 1):
                x = synth.gen_item(layers, H, T, D, d, kind, dtype=wl["dtype"])
                self.blobs[2 * d + kind] = ost.encode_item(x, self.schemes[2 * d + kind], self.lay)

    def run_once(self) -> tuple[int, float]:
        t0 = time.perf_counter()
        dec = {i: self.ost.decode_item(b, self.schemes[i], self.lay) for i, b in self.blobs.items()}
        K, V = self.ost.assemble(dec, self.req, self.lay)
        return K.nbytes + V.nbytes, time.perf_counter() - t0

    def describe(self, reps: int, nbytes: int) -> str:
        wl = self.wl
        return (f"assemble (decode + scatter) of request 0 (k={wl['k']}) restricted to layer(s) 0..{self.layers - 1} "
                f"of {wl['L']} (all {wl['H']} heads), {reps} repetition(s), {nbytes / 1e6:.0f} MB of "
                f"{wl['dtype']} KV output; numpy, single-threaded")


def oracle_baseline(wl, req, budget_s: float = 10.0, layers: int = 2):
    smp = OracleSample(wl, req, layers)
    total_b, total_t, reps = 0, 0.0, 0
    while reps < 1 or (total_t < budget_s and reps < 5):
        b, t = smp.run_once()
        total_b, total_t, reps = total_b + b, total_t + t, reps + 1
    return {"value": round(total_b / total_t / 1e9, 5), "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": smp.describe(reps, total_b)}


def run_reference(args, wl):
    """--impl reference: the CPU oracle as it stands, on rank 0 only."""
    if env_int("RANK", 0) != 0:
        return
    import synth
    reqs = synth.gen_requests(wl["n_docs"], wl["batch"], wl["k"], wl["s"], seed=1)
    smp = OracleSample(wl, reqs[0], layers=1)
    for _ in range(args.warmup):
        smp.run_once()
    times, nb = [], 0
    t0 = time.perf_counter()
    for _ in range(args.steps):
        b, t = smp.run_once()
        times.append(t)
        nb = b
        if time.perf_counter() - t0 > 150:  # keep the whole arm within a few minutes
            break
    tot = sum(times)
    v = nb * len(times) / tot / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": round(v, 5), "unit": "GB/s", "n_gpus": args.gpus,
            "steps": len(times), "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 2),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic",
            "config": {"workload": wl["desc"], "global_batch": wl["batch"], "k": wl["k"],
                       "step": "one bounded sample: " + smp.describe(1, nb)},
            "cpu_baseline": {"value": round(v, 5), "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": smp.describe(len(times), nb * len(times))},
            "e2e": {"value": round(v, 5), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# --------------------------------------------------------------------- ours
def run_ours(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2510_20878_b200 as hr
    import synth
    from paper_2510_20878_b200 import SCHEMES

    world = env_int("WORLD_SIZE", 1)
    rank = env_int("RANK", 0)
    local = env_int("LOCAL_RANK", 0)
    if args.gpus != world:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch N>1 with torchrun")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    L, H, D, T, k, B = wl["L"], wl["H"], wl["D"], wl["T"], wl["k"], wl["batch"]
    if H % world:
        raise SystemExit(f"H={H} not divisible by {world} GPUs")
    stream = torch.cuda.current_stream()

    # ---- inputs: hotness profile (offline) and request batches
    prof = synth.gen_requests(wl["n_docs"], 4 * wl["n_docs"], k, wl["s"], seed=7)
    h = hr.policy_count(prof, wl["n_docs"]).astype(np.uint64)
    n_batches = 8
    pool = synth.gen_requests(wl["n_docs"], n_batches * B, k, wl["s"], seed=1).reshape(n_batches, B, k)

    schemes = hr.policy_assign(h, wl["ladder"], wl["taus"])
    cfg = dict(L=L, H=H, D=D, T=T, dtype=wl["dtype"], ladder=wl["ladder"], taus=wl["taus"], rank=rank,
               world=world, device=local, keep_backing=False, decay_shift=1)
    total = sum(hr.item_bytes(int(s), **{k2: cfg[k2] for k2 in ("L", "H", "D", "T", "dtype", "rank", "world")})
                for s in schemes)
    st = hr.Store(hbm_budget=total + (1 << 20), **cfg)

    def src(doc, kp, vp, strm):
        synth.gen_item_device(kp, L, H, T, D, doc, 0, dtype=wl["dtype"], stream=strm)
        synth.gen_item_device(vp, L, H, T, D, doc, 1, dtype=wl["dtype"], stream=strm)

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    st.build(wl["n_docs"], h, src, stream=stream)
    build_s = time.perf_counter() - t0

    # ---- outputs: one [L][Hl][k*T][D] K and V buffer per request
    kvb = st.kv_bytes(k)
    out = torch.empty(2 * B * kvb // 2, dtype=torch.int16, device="cuda")
    ko = [out[(2 * r) * kvb // 2:(2 * r + 1) * kvb // 2] for r in range(B)]
    vo = [out[(2 * r + 1) * kvb // 2:(2 * r + 2) * kvb // 2] for r in range(B)]

    def step(i):
        st.assemble(pool[i % n_batches], ko, vo, stream=stream)
        if args.epoch_every and (i + 1) % args.epoch_every == 0:
            if world > 1:
                dist.all_reduce(st.hotness_delta(), op=dist.ReduceOp.SUM)
            st.replace(stream=stream)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
            torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    st.reset_stats()
    st.set_timing(True)
    sampler = clocks_sampler(local)
    time.sleep(0.1)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier()
    ev0.record(stream)
    for i in range(args.steps):
        step(args.warmup + i)
    ev1.record(stream)
    barrier()
    clocks = clocks_summary(*sampler)
    st.set_timing(False)
    ms = ev0.elapsed_time(ev1)
    stats = st.stats()
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda")
    bytes_t = torch.tensor([float(stats["bytes_out"])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
        dist.all_reduce(bytes_t, op=dist.ReduceOp.SUM)
    ms_max = float(ms_t.item())
    value = float(bytes_t.item()) / (ms_max / 1e3) / 1e9

    # ---- roofline of the dominant kernel (assemble_kv_kernel), live CUDA events
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except OSError:
        pass
    peak = peaks.get("hbm_gbs", 6650.0)
    peak_src = "MEASURED_PEAKS.json hbm_gbs (copy, read+write)" if "hbm_gbs" in peaks else "B200_PROFILING.md fallback"
    launches = max(1, stats["timed_launches"])
    avg_ms = stats["kernel_ms"] / launches
    alg_per_launch = stats["bytes_hbm_alg"] / max(1, stats["kernel_launches"])
    achieved = alg_per_launch / (avg_ms / 1e3) / 1e9
    traffic = args.ncu_traffic
    tfile = os.path.join(ROOT, "profiles", f"traffic_{args.workload}_b{B}_n{world}.json")
    if traffic is None and os.path.exists(tfile):
        with open(tfile) as f:
            traffic = json.load(f).get("dram_bytes_per_launch")
    roof = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
            "frac": round(achieved / peak, 4), "traffic": traffic, "kernel": "assemble_kv_kernel",
            "avg_launch_ms": round(avg_ms, 4), "alg_bytes_per_launch": int(alg_per_launch),
            "peak_source": peak_src}

    # ---- per-request assemble latency (one request, k docs, all HBM-resident)
    lat = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for i in range(min(64, n_batches * B)):
        req = pool.reshape(-1, k)[i:i + 1]
        e0.record(stream)
        st.assemble(req, ko[:1], vo[:1], stream=stream)
        e1.record(stream)
        e1.synchronize()
        lat.append(e0.elapsed_time(e1) * 1e3)
    lat_t = torch.tensor([float(np.percentile(lat, 50)), float(np.percentile(lat, 99))], device="cuda",
                         dtype=torch.float64)
    if world > 1:
        dist.all_reduce(lat_t, op=dist.ReduceOp.MAX)

    # ---- e2e through the C ABI with HOST buffers: ids from host, KV back to pinned host memory
    e2e = None
    if not args.no_e2e:
        host_out = [torch.empty(kvb // 2, dtype=torch.int16, pin_memory=True) for _ in range(4)]
        e2e_steps = max(1, min(3, args.steps))
        barrier()
        t_e0, t_e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t_e0.record(stream)
        d2h = 0
        for i in range(e2e_steps):
            ids = pool[i % n_batches]
            st.assemble(ids, ko, vo, stream=stream)
            for r in range(B):
                for j, src_t in enumerate((ko[r], vo[r])):
                    host_out[(2 * r + j) % 4].copy_(src_t, non_blocking=True)
                    d2h += kvb
        t_e1.record(stream)
        barrier()
        e2e_ms = torch.tensor([t_e0.elapsed_time(t_e1)], dtype=torch.float64, device="cuda")
        if world > 1:
            dist.all_reduce(e2e_ms, op=dist.ReduceOp.MAX)
        e2e_bytes = 2 * B * kvb * e2e_steps * world
        e2e = {"value": round(e2e_bytes / (float(e2e_ms.item()) / 1e3) / 1e9, 2), "unit": "GB/s",
               "h2d_bytes_per_step": int(B * k * 4 + 2 * B * k * 40), "d2h_bytes_per_step": int(d2h // e2e_steps),
               "path": "hr_assemble_kv(host ids) -> device KV -> cudaMemcpyAsync D2H into pinned host buffers"}

    # ---- build (a2-a5) throughput, reported beside the step
    src_bytes = wl["n_docs"] * 2 * L * (H // world) * T * D * 2
    build = {"seconds": round(build_s, 3), "source_GBps_incl_generation": round(src_bytes / build_s / 1e9, 2),
             "items": 2 * wl["n_docs"]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = oracle_baseline(wl, pool[0][0], budget_s=10.0, layers=2)

    sch_hist = {name: int(np.sum(schemes == code)) for name, code in SCHEMES.items() if np.sum(schemes == code)}
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms_max / args.steps, 4), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": wl["dtype"], "data": "synthetic",
        "config": {"workload": wl["desc"], "global_batch": B, "k": k, "seq_len_per_request": k * T,
                   "parallelism": f"kv-head shard x{world}" if world > 1 else "single GPU",
                   "n_docs": wl["n_docs"], "items_per_scheme": sch_hist, "epoch_every_steps": args.epoch_every,
                   "l2": "inputs larger than L2 (store and per-step output each >> 126 MB)",
                   "store_bytes_per_rank": int(total)},
        "request_latency_us": {"p50": round(lat_t[0].item(), 1), "p99": round(lat_t[1].item(), 1),
                               "k": k, "bytes_out": int(2 * kvb)},
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "gpu_launches": int(stats["kernel_launches"]),
        "clocks": clocks,
        "build": build,
        "impl": "ours",
    }
    if rank == 0:
        print(json.dumps(line), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--epoch-every", type=int, default=8)
    ap.add_argument("--batch", type=int, default=0, help="override the workload's batch (profiling runs)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ncu-traffic", type=float, default=None,
                    help="dram read+write bytes per launch from an ncu --set full capture (profiles/)")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "ours":
        raise SystemExit("--warmup must be >= 3")
    wl = dict(WORKLOADS[args.workload])
    if args.batch:
        wl["batch"] = args.batch
    if args.impl == "reference":
        run_reference(args, wl)
    else:
        run_ours(args, wl)


if __name__ == "__main__":
    main()
