"""Pinned H2D bandwidth vs the NUMA placement of the pinned buffer: the GPU's PCI
device NUMA node / local CPUs, then 52.7 MB H2D with the process bound to each node's
CPUs before the pinned allocation (first touch places the pages)."""
import os
import subprocess
import sys

import torch


def gpu_pci():
    bdf = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
                         text=True).stdout.strip().splitlines()[0].lower()
    dom, rest = bdf.split(":", 1)
    return f"{int(dom, 16):04x}:{rest}"


def node_cpus():
    out = {}
    base = "/sys/devices/system/node"
    for d in sorted(os.listdir(base)):
        if d.startswith("node") and d[4:].isdigit():
            cl = open(f"{base}/{d}/cpulist").read().strip()
            cpus = set()
            for part in cl.split(","):
                if "-" in part:
                    a, b = part.split("-")
                    cpus.update(range(int(a), int(b) + 1))
                elif part:
                    cpus.add(int(part))
            out[int(d[4:])] = cpus
    return out


def bw(n_bytes=52_699_000, reps=10):
    n = n_bytes // 4
    h = torch.empty(n, dtype=torch.float32).pin_memory()
    h.fill_(1.0)
    d = torch.empty(n, dtype=torch.float32, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    return n * 4 / (a.elapsed_time(b) / reps) / 1e6


if __name__ == "__main__":
    if len(sys.argv) > 1:  # child: bind to node, allocate, measure
        node = int(sys.argv[1])
        os.sched_setaffinity(0, node_cpus()[node])
        torch.cuda.init()
        print(f"node {node}: {bw():.1f} GB/s", flush=True)
        sys.exit(0)
    pci = gpu_pci()
    try:
        gnode = open(f"/sys/bus/pci/devices/{pci}/numa_node").read().strip()
        lcpu = open(f"/sys/bus/pci/devices/{pci}/local_cpulist").read().strip()
    except OSError as e:
        gnode, lcpu = f"? ({e})", "?"
    nodes = node_cpus()
    print(f"gpu {pci} numa_node {gnode} local_cpulist {lcpu}; nodes {[(k, len(v)) for k, v in nodes.items()]}")
    print(f"unbound: {bw():.1f} GB/s", flush=True)
    for k in nodes:
        subprocess.run([sys.executable, __file__, str(k)])
