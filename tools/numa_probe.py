"""H2D bandwidth of pinned host memory vs the NUMA node the pinning thread runs on
(first-touch placement): the GPU's node from sysfs, then one 2 GB copy per node."""
import glob
import os
import subprocess

import torch

torch.cuda.init()
bdf = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader"], capture_output=True,
                     text=True).stdout.strip().splitlines()[0].lower()
bdf = bdf[4:] if len(bdf) > 12 else bdf  # 00000000:xx:yy.z -> 0000:xx:yy.z
try:
    gnode = open(f"/sys/bus/pci/devices/{bdf}/numa_node").read().strip()
except OSError as e:
    gnode = f"? ({e})"
print("gpu", bdf, "numa_node", gnode, "cpus allowed", len(os.sched_getaffinity(0)))
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
allowed = os.sched_getaffinity(0)
dst = torch.empty(2 << 30, dtype=torch.uint8, device="cuda")


def parse(s):
    out = set()
    for part in s.strip().split(","):
        if "-" in part:
            a, b = part.split("-")
            out |= set(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


for nd in nodes:
    cpus = parse(open(nd + "/cpulist").read()) & allowed
    if not cpus:
        print(os.path.basename(nd), "no allowed cpus")
        continue
    os.sched_setaffinity(0, cpus)
    src = torch.empty(2 << 30, dtype=torch.uint8)
    src.fill_(1)  # first touch on this node
    src = src.pin_memory()
    best = 0.0
    for _ in range(4):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        dst.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, src.numel() / (e0.elapsed_time(e1) * 1e-3) / 1e9)
    print(os.path.basename(nd), f"cpus {min(cpus)}-{max(cpus)} ({len(cpus)}): H2D {best:.1f} GB/s", flush=True)
    del src
    os.sched_setaffinity(0, allowed)
