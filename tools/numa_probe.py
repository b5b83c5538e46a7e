"""Does the page-locked D2H rate depend on the NUMA node of the host buffer?
Prints the GPU's NUMA node, the host topology, and the 128 MiB D2H rate with the
process bound to each node's CPUs (first touch places the buffer there)."""
import glob
import os
import subprocess
import time

import torch

print(subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout)
bus = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
print("pci", bus)
for p in glob.glob("/sys/bus/pci/devices/*/numa_node"):
    try:
        cls = open(os.path.dirname(p) + "/class").read().strip()
        if cls.startswith("0x0302") or cls.startswith("0x0300"):
            print(p, open(p).read().strip())
    except OSError:
        pass
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes", [(os.path.basename(n), open(n + "/cpulist").read().strip()) for n in nodes])
print("affinity now", sorted(os.sched_getaffinity(0)))


def parse(cl):
    out = set()
    for part in cl.split(","):
        if "-" in part:
            a, b = part.split("-")
            out |= set(range(int(a), int(b) + 1))
        elif part:
            out.add(int(part))
    return out


dev = torch.empty(32 << 20, dtype=torch.int32, device="cuda")
allowed = os.sched_getaffinity(0)
for n in nodes:
    cpus = parse(open(n + "/cpulist").read().strip()) & allowed
    if not cpus:
        print(os.path.basename(n), "no allowed cpus")
        continue
    os.sched_setaffinity(0, cpus)
    host = torch.empty(32 << 20, dtype=torch.int32).pin_memory()
    host.zero_()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(5):
        t = time.perf_counter()
        host.copy_(dev, non_blocking=True)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    print(os.path.basename(n), f"D2H 128 MiB: {best * 1e3:.2f} ms = {0.134217728 / best:.1f} GB/s")
    del host
os.sched_setaffinity(0, allowed)
