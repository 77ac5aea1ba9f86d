#!/usr/bin/env python
"""Benchmark of the S2 sparse-sketch reduce on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--config resnet50]

One step = one full reduce of one synthetic gradient per rank: compress (bitmap +
compaction + count-sketch insert) -> sketch all-reduce + bitmap all-gather/OR
(N > 1, NCCL over NVLink) -> median decode (÷N) into a dense fp32 gradient.

Prints ONE JSON line (rank 0).  ``value`` = dense-equivalent GB/s reduced per GPU
= 4*d / t_reduce (BASELINE.json's metric; t = max over ranks, CUDA events, K steps);
``job_GBps`` = N * 4*d / t_reduce, the whole job; ``ms_per_step`` = t_reduce.  ``e2e`` repeats the measurement through the same C-ABI call with
pinned HOST buffers, H2D of the gradient and D2H of the result inside the timed
region.  ``--impl reference`` times the CPU reference path (the NumPy oracle
port of sketchgrad.sparse, bit-identical to the as-shipped reference) on all the
host cores instead (oracle/parallel.py).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "dense-equivalent gradient GB/s reduced per GPU and ms/reduce at 1/2/4/8 B200"
CONFIGS = {
    # configs[1] of BASELINE.json: the headline (fits one GPU)
    "resnet50": dict(dim=25_600_000, alpha=0.01, rows=3, cols=262_144, label="ResNet-50-sized 25.6M fp32, 99% sparse"),
    "bert": dict(dim=110_000_000, alpha=0.05, rows=5, cols=1_048_576, label="BERT-base-sized 110M fp32, 95% sparse"),
    "bert_np2": dict(dim=110_000_000, alpha=0.05, rows=5, cols=1_000_000, label="BERT-base 110M, 95%, 5x1,000,000"),
    "lstm": dict(dim=200_000_000, alpha=0.001, rows=3, cols=1_048_576, grid=(200_000, 1_000),
                 label="LSTM-LM embedding 200M fp32 (200k x 1000), 99.9% row-sparse, element bitmap"),
    "lstm_rows": dict(dim=200_000_000, alpha=0.001, rows=3, cols=1_048_576, grid=(200_000, 1_000),
                      num_blocks=200_000, label="LSTM-LM embedding 200M, 99.9% row-sparse, row bitmap (b=200k)"),
    "lstm_rows_zipf": dict(dim=200_000_000, alpha=0.001, rows=3, cols=1_048_576, grid=(200_000, 1_000),
                           num_blocks=200_000, zipf=1.1,
                           label="LSTM-LM embedding 200M, 99.9% Zipf(1.1) rows (ranks overlap), row bitmap"),
    "gpt2m_90": dict(dim=355_000_000, alpha=0.10, rows=3, cols=1_048_576, label="GPT-2-medium 355M, 90% sparse"),
    "gpt2m_99": dict(dim=355_000_000, alpha=0.01, rows=3, cols=1_048_576, label="GPT-2-medium 355M, 99% sparse"),
    "gpt2m_999": dict(dim=355_000_000, alpha=0.001, rows=3, cols=262_144, label="GPT-2-medium 355M, 99.9% sparse"),
    # union densities a W=2 / W=4 reduce decodes (dev configs for single-GPU decode tuning)
    "resnet50_d2": dict(dim=25_600_000, alpha=0.02, rows=3, cols=262_144, label="ResNet-50-sized, 98% sparse"),
    "resnet50_d4": dict(dim=25_600_000, alpha=0.04, rows=3, cols=262_144, label="ResNet-50-sized, 96% sparse"),
    # 1 - 0.99^8: the union a W = 8 reduce decodes (single-GPU proxy for the north-star W = 8 decode)
    "resnet50_d8": dict(dim=25_600_000, alpha=0.0773, rows=3, cols=262_144, label="ResNet-50-sized, 92.3% sparse"),
    "oracle1m": dict(dim=1_000_000, alpha=0.01, rows=3, cols=16_384, label="1M fp32, 99% sparse (configs[0])"),
}
N_ROTATE = 4  # distinct gradient buffers cycled through: N_ROTATE * 4d bytes > 126 MB L2
HBM_FALLBACK = 6650.0  # GB/s, B200_PROFILING.md fallback


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return HBM_FALLBACK, "fallback"


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled in the background (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None
        self.marks = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index),
                 "--query-gpu=timestamp,clocks.sm,clocks.max.sm,power.draw,utilization.gpu,"
                 "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append((time.time(), [x.strip() for x in line.split(",")]))

    def mark(self, name):
        self.marks.append((name, time.time()))

    def stop(self):
        if self.proc is None:
            return None
        time.sleep(0.12)
        self.proc.terminate()
        try:
            self.proc.wait(2)
        except Exception:
            self.proc.kill()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        marks = dict(self.marks)
        t0, t1 = marks.get("load_start", 0), marks.get("load_end", time.time())
        sm, mx, reasons, in_load = [], 0.0, set(), 0
        for ts, r in self.rows:
            try:
                smv, mxv = float(r[1]), float(r[2])
            except (ValueError, IndexError):
                continue
            mx = max(mx, mxv)
            if t0 <= ts <= t1:
                in_load += 1
                sm.append(smv)
                for n, v in zip(names, r[5:9]):
                    if v.lower() == "active":
                        reasons.add(n)
        if not sm:  # region shorter than the sampling period: use every sample of the run
            for ts, r in self.rows:
                try:
                    sm.append(float(r[1]))
                except (ValueError, IndexError):
                    pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples_under_load": in_load, "samples": len(self.rows)}


# Measured ceilings of the two non-HBM resources the kernels can saturate (1 B200, this pool):
# random 4-byte L2 gathers — one L1->crossbar request per SM cycle, shared with every written
# 32-byte sector (profiles/r02_dsmem_bench.json "l2_gather", profiles/r02_ab_decode_bulk_qr.txt) —
# and random fp32 red.global.add into an L2-resident table (profiles/r02_atomics_bench.json).
L2_REQ_PER_S = 295.5e9
L2_RED_PER_S = 185.0e9
NVLINK_A2A_GBS = 646.0


def kernel_floors(d, rows, cols, words_bytes, nnz, union, hbm_peak):
    """Lower bounds on the compress / decode durations from the measured ceilings: HBM bytes at the
    copy peak; compress REDs (rows x nnz) at the L2 RED rate; decode L1->xbar requests (rows x union
    gathers + written output / next-table / bitmap sectors) at the request rate."""
    table_bytes = 4 * rows * cols
    hbm_c = (4 * d + words_bytes + table_bytes) / (hbm_peak * 1e9) * 1e6
    red_c = rows * nnz / L2_RED_PER_S * 1e6
    req = rows * union + (4 * d + table_bytes + words_bytes) / 32
    hbm_d = (4 * d + 2 * table_bytes + words_bytes) / (hbm_peak * 1e9) * 1e6
    req_d = req / L2_REQ_PER_S * 1e6
    return {
        "compress": {"us": round(max(hbm_c, red_c), 2), "bound": "hbm" if hbm_c >= red_c else "l2 red",
                     "hbm_us": round(hbm_c, 2), "red_us": round(red_c, 2), "reds": rows * nnz},
        "decode": {"us": round(max(hbm_d, req_d), 2), "bound": "hbm" if hbm_d >= req_d else "l1-xbar requests",
                   "hbm_us": round(hbm_d, 2), "request_us": round(req_d, 2), "requests": int(req),
                   "union": union},
    }


# ----------------------------------------------------------------- reference


def _host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def _ref_grads(cfg, W):
    from oracle import s2_oracle as o

    return [o.synthetic_gradient(cfg["dim"], cfg["alpha"], r) if cfg.get("grid") is None
            else _rows_gradient_np(cfg, r) for r in range(W)]


def _time_reference(cfg, W, warmup, max_steps, budget_s):
    """Oracle port of sketchgrad.sparse on every host core (oracle/parallel.py): W ranks'
    compress, merge, decompress per step.  Returns (s/step, steps, cores)."""
    from oracle.parallel import ParallelReference

    pr = ParallelReference(_ref_grads(cfg, W), cfg["rows"], cfg["cols"], 0, procs=_host_cores(),
                           num_blocks=cfg.get("num_blocks", cfg["dim"]))
    try:
        for _ in range(warmup):
            pr.step()
        t0, done = time.perf_counter(), 0
        while done < max_steps:
            pr.step()
            done += 1
            if time.perf_counter() - t0 > budget_s and done >= 3:
                break  # bounded sample: the run must finish within a few minutes
        return (time.perf_counter() - t0) / done, done, pr.procs
    finally:
        pr.close()


def reference_arm(args, cfg):
    """CPU reference on the host cores, rank 0 only under torchrun."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = args.gpus
    d = cfg["dim"]
    dt, done, cores = _time_reference(cfg, W, args.warmup, args.steps, args.ref_budget)
    value = 4 * d / dt / 1e9  # per GPU: each step reduces W ranks' d-element gradients
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "job_GBps": round(W * value, 4),
        "unit": "GB/s", "n_gpus": W,
        "steps": done, "warmup": args.warmup, "ms_per_step": round(dt * 1e3, 3),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": _config_json(args, cfg),
        "cpu_baseline": {"value": round(value, 4), "unit": "GB/s", "cores": cores, "kind": "port",
                         "sample": f"full workload per step: {W} ranks' compress + merge + decompress of "
                                   f"{d} elements each, chunked over {cores} worker processes "
                                   f"(oracle/parallel.py); numpy {np.__version__}"},
        "e2e": {"value": round(value, 4), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def cpu_baseline(cfg, budget_s=10.0):
    """Oracle port timed on this host's cores (rank 0, N=1): compress + merge + decompress of one
    gradient; plus the reference's call structure as shipped (single-threaded NumPy, Python slice
    loops for index extraction) at configs[0] = 1M / 99 % / 3 x 16384."""
    dt, n, cores = _time_reference(cfg, 1, 1, 50, budget_s)
    out = {"value": round(4 * cfg["dim"] / dt / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "port",
           "sample": f"{n} full reduces (W=1) of the {cfg['dim']}-element workload, chunked over {cores} "
                     f"worker processes (oracle/parallel.py); numpy {np.__version__}"}
    from oracle import s2_oracle as o

    c0 = CONFIGS["oracle1m"]
    g = o.synthetic_gradient(c0["dim"], c0["alpha"], 0)
    o.reduce_as_shipped([g], c0["rows"], c0["cols"], 0)  # warm-up
    t0, k = time.perf_counter(), 0
    while k < 3 or (time.perf_counter() - t0 < 5.0 and k < 20):
        o.reduce_as_shipped([g], c0["rows"], c0["cols"], 0)
        k += 1
    dts = (time.perf_counter() - t0) / k
    out["as_shipped"] = {"value": round(4 * c0["dim"] / dts / 1e9, 5), "unit": "GB/s", "ms_per_step": round(dts * 1e3, 1),
                         "cores": 1, "kind": "port-as-shipped",
                         "sample": f"{k} reduces (W=1) of configs[0] (1M fp32, 99 % sparse, 3x16384) through "
                                   "oracle.reduce_as_shipped: the reference's call structure incl. its Python "
                                   "slice loops (core.py:195-200, sparse.py:44-49), one process, one core"}
    return out


def _rows_gradient_np(cfg, rank=0):
    V, H = cfg["grid"]
    rng = np.random.default_rng(1234 + rank)
    p = None
    if cfg.get("zipf"):
        from paper_2110_02140_b200.synthetic import zipf_weights

        p = zipf_weights(V, cfg["zipf"])
    r = rng.choice(V, max(1, int(round(cfg["alpha"] * V))), replace=False, p=p)
    g = np.zeros(cfg["dim"], dtype=np.float32)
    for row in r:
        g[row * H:(row + 1) * H] = rng.standard_normal(H).astype(np.float32)
    return g


def _config_json(args, cfg):
    return {"workload": f"{args.config}: {cfg['label']}, sketch {cfg['rows']}x{cfg['cols']}, W={args.gpus}",
            "dim": cfg["dim"], "nnz_per_rank": int(round(cfg["alpha"] * cfg["dim"])), "rows": cfg["rows"],
            "cols": cfg["cols"], "world": args.gpus, "parallelism": f"dp{args.gpus}",
            "num_blocks": cfg.get("num_blocks", cfg["dim"]),
            "pipeline": args.pipeline if args.gpus > 1 else 1,
            "l2": f"inputs rotate over {N_ROTATE if cfg['dim'] <= 50_000_000 else 2} gradient buffers "
                  f"({(N_ROTATE if cfg['dim'] <= 50_000_000 else 2) * 4 * cfg['dim'] / 1e6:.0f} MB > 126 MB L2)"}


# --------------------------------------------------------------------- ours


def ours(args, cfg):
    import ctypes

    import torch
    import torch.distributed as dist

    world = args.gpus
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2110_02140_b200 as s2
    from paper_2110_02140_b200 import synthetic
    from paper_2110_02140_b200._lib import check, lib, ptr

    d, rows, cols = cfg["dim"], cfg["rows"], cfg["cols"]
    red = s2.S2Reducer(d, rows=rows, cols=cols, seed=0, world=world, rank=rank, num_blocks=cfg.get("num_blocks"))
    gcfg = dict(dim=d, alpha=cfg["alpha"], rows=cfg.get("grid"), zipf=cfg.get("zipf"))
    n_rot = N_ROTATE if d <= 50_000_000 else 2  # 2 x >= 440 MB still exceeds the 126 MB L2
    grads = [synthetic.gradient(gcfg, rank, base_seed=1234 + 1000 * k) for k in range(n_rot)]
    outs = [torch.empty(d, dtype=torch.float32, device="cuda") for _ in range(n_rot)]
    stream = torch.cuda.current_stream()
    sp = ctypes.c_void_p(stream.cuda_stream)
    h = red.plan.handle
    gp = [ptr(g) for g in grads]
    op = [ptr(x) for x in outs]
    null = ctypes.c_void_p(0)

    def step(i):
        check(lib.s2_reduce(h, gp[i % n_rot], op[i % n_rot], null, sp))

    # pipelined batches (s2_reduce_many, W > 1): compress of step k+1 beside step k's exchange
    P = max(1, args.pipeline if world > 1 else 1)
    batches = {}

    def batch(i, n):
        key = (i % n_rot, n)
        if key not in batches:
            batches[key] = ((ctypes.c_void_p * n)(*[gp[(i + k) % n_rot] for k in range(n)]),
                            (ctypes.c_void_p * n)(*[op[(i + k) % n_rot] for k in range(n)]))
        g_arr, o_arr = batches[key]
        check(lib.s2_reduce_many(h, g_arr, o_arr, n, sp))

    def run(n_steps, i0=0):
        if P == 1:
            for i in range(i0, i0 + n_steps):
                step(i)
            return
        for i in range(i0, i0 + n_steps, P):
            batch(i, min(P, i0 + n_steps - i))

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    clocks = ClockSampler(local)
    clocks.start()
    time.sleep(0.2)
    clocks.mark("load_start")
    for i in range(args.warmup):
        step(i)
    # soak (extra untimed warm-up): keep the GPU busy until clocks and memory power states settle —
    # at least 0.5 s and until two consecutive 50-step batches agree within 2 % (at most 3 s; a
    # fresh box's first run once measured 45 % slow after a fixed 0.3 s soak)
    barrier()
    t_soak = time.time()
    i, prev = 0, None
    sa, sb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while True:
        sa.record(stream)
        for _ in range(50):
            step(i)
            i += 1
        sb.record(stream)
        torch.cuda.synchronize()
        cur = sa.elapsed_time(sb)
        settled = prev is not None and abs(cur - prev) <= 0.02 * prev
        prev = cur
        done = time.time() - t_soak > 0.5 and settled
        if world > 1:  # every rank leaves the soak together
            flag = torch.tensor([0.0 if done or time.time() - t_soak > 3.0 else 1.0], device="cuda")
            dist.all_reduce(flag, op=dist.ReduceOp.MAX)
            if flag.item() == 0.0:
                break
        elif done or time.time() - t_soak > 3.0:
            break
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms_plain = None
    if P > 1:  # latency view: the same steps one reduce at a time
        e0.record(stream)
        for i in range(args.steps):
            step(i)
        e1.record(stream)
        barrier()
        ms_plain = max_over_ranks(e0.elapsed_time(e1) / args.steps)
        run(2 * P)  # warm the pipelined path
        barrier()
    e0.record(stream)
    th0 = time.perf_counter()
    run(args.steps)
    host_us = (time.perf_counter() - th0) / args.steps * 1e6  # host enqueue cost per step
    e1.record(stream)
    barrier()
    ms = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    host_us = max_over_ranks(host_us)

    # per-phase durations: the same s2_reduce launches with the plan's timing events
    # (recorded on the launching stream between compress / aggregate / decode)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    for e in ev:
        e.record(stream)
    evs = (ctypes.c_void_p * 4)(*[e.cuda_event for e in ev])
    check(lib.s2_plan_set_timing_events(h, evs, 4))
    phases = {"compress": 0.0, "aggregate": 0.0, "decode": 0.0}
    nph = max(args.steps, 20)
    barrier()
    for i in range(nph):
        step(i)
        ev[3].synchronize()
        phases["compress"] += ev[0].elapsed_time(ev[1])
        phases["aggregate"] += ev[1].elapsed_time(ev[2])
        phases["decode"] += ev[2].elapsed_time(ev[3])
    check(lib.s2_plan_set_timing_events(h, None, 0))
    phases = {k: max_over_ranks(v / nph) for k, v in phases.items()}
    # union coordinates the decode queried (non-zeros of a decoded output; an exactly-zero
    # median of real-valued estimates does not occur at these sizes)
    union = int(max_over_ranks(float((outs[0] != 0).sum().item())))
    del outs

    # e2e: pinned host gradient in, pinned host result out, every step's H2D and D2H inside the
    # timed region; HostPipeline overlaps step i's reduce with step i+1's H2D and i-1's D2H
    from paper_2110_02140_b200.reducer import HostPipeline

    hg = [torch.empty(d, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    for k in range(2):
        hg[k].copy_(grads[k].cpu())
    ho = [torch.empty(d, dtype=torch.float32, pin_memory=True) for _ in range(2)]
    pipe = HostPipeline(red)
    ke = max(3, min(args.steps, 50))
    for i in range(3):
        pipe.submit(hg[i % 2], ho[i % 2])
    pipe.drain()
    barrier()
    e0.record(pipe.s_in)  # device timing: first H2D start ... last D2H end
    for i in range(ke):
        pipe.submit(hg[i % 2], ho[i % 2])
    e1.record(pipe.s_out)
    pipe.drain()
    torch.cuda.synchronize()
    ms_e2e = max_over_ranks(e0.elapsed_time(e1) / ke)
    barrier()

    # side-by-side: dense NCCL all-reduce of the same fp32 gradient, the
    # uncompressed exchange a DDP step would do instead of the sparse-sketch reduce
    dense = None
    if world > 1:
        buf = grads[0].clone()
        kd = max(5, min(args.steps, 50))
        for _ in range(5):
            dist.all_reduce(buf)
        barrier()
        e0.record(stream)
        for _ in range(kd):
            dist.all_reduce(buf)
        e1.record(stream)
        barrier()
        ms_dense = max_over_ranks(e0.elapsed_time(e1) / kd)
        dense = {"ms_per_step": round(ms_dense, 5), "value": round(4 * d / (ms_dense * 1e-3) / 1e9, 2),
                 "unit": "GB/s", "op": f"torch.distributed.all_reduce (NCCL, SUM) of {d} fp32, device-resident"}
        del buf
    barrier()
    clocks.mark("load_end")
    clk = clocks.stop()

    red.check_finite()
    red.check_exchange()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    hbm_peak, peak_kind = peaks()
    B = 4 * d
    words_bytes = 4 * (-(-cfg.get("num_blocks", d) // 32))
    table_bytes = 4 * rows * cols
    alg = {"compress": B + words_bytes + table_bytes, "decode": words_bytes + table_bytes + B}
    dom = max(("compress", "decode"), key=lambda k: phases[k])
    ach = alg[dom] / (phases[dom] * 1e-3) / 1e9
    traffic, ncu = None, None
    tfile = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tfile):
        tj = json.load(open(tfile))
        traffic = tj.get(f"{args.config}:{dom}")
        # the same kernel's duration from the committed ncu launch list (cold L2, serialised)
        nd = tj.get(f"{args.config}:{dom}:ncu_us")
        if nd:
            na = alg[dom] / (nd * 1e-6) / 1e9
            ncu = {"us": nd, "achieved": round(na, 1), "frac": round(na / hbm_peak, 4),
                   "source": tj.get("_source", "profiles/traffic.json")}
    phase_out = {}
    nnz = int(round(cfg["alpha"] * (cfg["grid"][0] if cfg.get("grid") else d))) * (cfg["grid"][1] if cfg.get("grid") else 1)
    floors = kernel_floors(d, rows, cols, words_bytes, nnz, union, hbm_peak)
    for k in ("compress", "decode"):
        a = alg[k] / (phases[k] * 1e-3) / 1e9
        fl = floors[k]
        phase_out[k] = {"ms": round(phases[k], 5), "GB/s": round(a, 1), "frac": round(a / hbm_peak, 4),
                        "algorithmic_bytes": alg[k],
                        "floor": dict(fl, frac=round(fl["us"] / (phases[k] * 1e3), 4))}
    if world > 1:
        bus = 2 * (world - 1) / world * table_bytes + (world - 1) / world * world * words_bytes
        bus_gbs = bus / (phases["aggregate"] * 1e-3) / 1e9
        phase_out["aggregate"] = {"ms": round(phases["aggregate"], 5), "bus_GB/s": round(bus_gbs, 1),
                                  "bus_bytes": bus, "frac_of_900": round(bus_gbs / 900.0, 4),
                                  "frac_of_measured": round(bus_gbs / NVLINK_A2A_GBS, 4),
                                  "measured_peak": f"{NVLINK_A2A_GBS} GB/s: all-to-all SM stores, 32 MiB per peer, "
                                                   "W=4 (profiles/r02_nvlink_bench_w4.json)"}
    value = B / (ms * 1e-3) / 1e9  # per GPU (BASELINE.json metric); job_GBps = world * value
    line = {
        "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(ms, 5), "job_GBps": round(world * value, 2),
        "latency_ms_per_reduce": round(ms_plain if ms_plain is not None else ms, 5),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": _config_json(args, cfg),
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": round(ach, 1), "peak": hbm_peak, "unit": "GB/s",
                     "frac": round(ach / hbm_peak, 4), "traffic": traffic, "peak_kind": peak_kind,
                     "bytes_per_launch": alg[dom], "timing": "CUDA events around the kernel inside the step",
                     "ncu": ncu, "measured_floor": phase_out[dom]["floor"]},
        "phases": phase_out,
        "e2e": {"value": round(B / (ms_e2e * 1e-3) / 1e9, 3), "unit": "GB/s", "ms_per_step": round(ms_e2e, 4),
                "h2d_bytes_per_step": B, "d2h_bytes_per_step": B,
                "path": "HostPipeline.submit -> S2Reducer.reduce (C-ABI s2_reduce); pinned host buffers; "
                        "H2D/D2H of every step inside the timed region (CUDA events: first H2D start to "
                        "last D2H end; copies overlapped across steps on separate streams)"},
        "gpu_launches": args.steps * (3 if world > 1 else 2),
        "host_enqueue_us_per_step": round(host_us, 2),
        "clocks": clk,
    }
    if dense is not None:
        line["dense_allreduce"] = dense
    if world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(cfg, args.cpu_budget)
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="resnet50", choices=sorted(CONFIGS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    ap.add_argument("--ref-budget", type=float, default=120.0, help="max seconds of timed reference steps")
    ap.add_argument("--alpha", type=float, default=None, help="override the config's non-zero fraction")
    ap.add_argument("--cols", type=int, default=None, help="override the config's sketch width")
    ap.add_argument("--pipeline", type=int, default=8,
                    help="W > 1: reduces per s2_reduce_many batch (1 = one s2_reduce per step)")
    args = ap.parse_args()
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    if ws != args.gpus and "WORLD_SIZE" in os.environ:
        args.gpus = ws
    args.warmup = max(args.warmup, 3)
    cfg = dict(CONFIGS[args.config])
    if args.alpha is not None:
        cfg["alpha"] = args.alpha
        cfg["label"] += f" (alpha={args.alpha})"
    if args.cols is not None:
        cfg["cols"] = args.cols
    if args.impl == "reference":
        reference_arm(args, cfg)
    else:
        ours(args, cfg)


if __name__ == "__main__":
    main()
