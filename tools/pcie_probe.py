"""Host<->device copy ceilings for the e2e path: per GPU, pinned 102 MB H2D, D2H and both
concurrently, with N GPUs copying at once, with and without binding each process (and its
pinned pages, first touch) to the GPU's local CPUs (/sys/bus/pci/devices/<bus>/local_cpulist).

    python tools/pcie_probe.py            # prints one JSON line per (n, affinity)
"""
import json
import multiprocessing as mp
import os
import sys


def local_cpus(dev: int):
    import subprocess

    bus = subprocess.run(["nvidia-smi", "-i", str(dev), "--query-gpu=pci.bus_id", "--format=csv,noheader"],
                         capture_output=True, text=True).stdout.strip().lower()
    if bus.startswith("0000000"):
        bus = bus[4:]
    path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
    if not os.path.exists(path):
        return None, bus
    cpus = set()
    for part in open(path).read().strip().split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus, bus


def worker(dev, affinity, nbytes, q, barrier):
    import torch

    torch.cuda.set_device(dev)
    cpus, bus = local_cpus(dev)
    if affinity and cpus:
        os.sched_setaffinity(0, cpus)
    n = nbytes // 4
    h_in = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_out = torch.empty(n, dtype=torch.float32, pin_memory=True)
    h_in.fill_(1.0)
    h_out.fill_(0.0)
    d_in = torch.empty(n, dtype=torch.float32, device="cuda")
    d_out = torch.empty(n, dtype=torch.float32, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    res = {"dev": dev, "bus": bus, "ncpus_local": len(cpus) if cpus else None}

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        barrier.wait()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(torch.cuda.current_stream())
        for _ in range(reps):
            fn()
        s1.synchronize()
        s2.synchronize()
        e1.record(torch.cuda.current_stream())
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    def h2d():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)

    def d2h():
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s2)

    def both():
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
        torch.cuda.current_stream().wait_stream(s1)
        torch.cuda.current_stream().wait_stream(s2)

    for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
        ms = timed(fn)
        res[name + "_ms"] = round(ms, 4)
        res[name + "_GBps"] = round(nbytes / (ms * 1e-3) / 1e9, 1)
    q.put(res)


def run(n, affinity, nbytes=102_400_000):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    barrier = ctx.Barrier(n)
    ps = [ctx.Process(target=worker, args=(d, affinity, nbytes, q, barrier)) for d in range(n)]
    for p in ps:
        p.start()
    out = [q.get() for _ in range(n)]
    for p in ps:
        p.join()
    return sorted(out, key=lambda r: r["dev"])


if __name__ == "__main__":
    import torch

    ng = torch.cuda.device_count()
    for n in sorted({1, ng}):
        for aff in (False, True):
            print(json.dumps({"n": n, "affinity": aff, "per_gpu": run(n, aff)}), flush=True)
    sys.exit(0)
