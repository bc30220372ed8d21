"""Does the NUMA node of the pinned staging buffers matter for the host->device->host path?
For every node: pin this thread to its CPUs, allocate pinned buffers (first touch there), time
1 GiB up and 1 GiB down at once on two streams.  usage: python tools/numa_probe.py"""
import glob, os, sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import paper_2012_08655_b200 as fk

def cpus(path):
    out = []
    for part in open(path).read().strip().split(","):
        if not part: continue
        a, _, b = part.partition("-")
        out += list(range(int(a), int(b or a) + 1))
    return out

bdf = torch.cuda.get_device_properties(0).pci_bus_id if hasattr(torch.cuda.get_device_properties(0), "pci_bus_id") else None
try:
    import ctypes
    buf = ctypes.create_string_buffer(32)
    torch.cuda.init()
    rt = ctypes.CDLL("libcudart.so.12")
    rt.cudaDeviceGetPCIBusId(buf, 32, 0)
    bdf = buf.value.decode().lower()
except Exception as e:
    print("bus id:", e)
node = None
for cand in (f"/sys/bus/pci/devices/{bdf}/numa_node",):
    if bdf and os.path.exists(cand):
        node = int(open(cand).read())
print("gpu", bdf, "numa_node", node, "cpu_count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
nodes = sorted(glob.glob("/sys/devices/system/node/node[0-9]*"))
print("nodes:", [(n.rsplit("node", 1)[1], len(cpus(n + "/cpulist"))) for n in nodes])
full = os.sched_getaffinity(0)
N = 1 << 30
d_in = torch.empty(N, dtype=torch.uint8, device="cuda"); d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
for n in nodes + ["all"]:
    if n == "all":
        os.sched_setaffinity(0, full)
    else:
        c = set(cpus(n + "/cpulist")) & full
        if not c: continue
        os.sched_setaffinity(0, c)
    h_in = fk.pinned_empty((N,), np.uint8); h_out = fk.pinned_empty((N,), np.uint8)
    h_in[:] = 1; h_out[:] = 0
    ti, to = torch.from_numpy(h_in), torch.from_numpy(h_out)
    best = 1e9
    for rep in range(4):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        with torch.cuda.stream(s1): d_in.copy_(ti, non_blocking=True)
        with torch.cuda.stream(s2): to.copy_(d_out, non_blocking=True)
        torch.cuda.synchronize(); best = min(best, time.perf_counter() - t0)
    print(f"node {n.rsplit('node', 1)[-1]:>4}: {N / best / 1e9:6.1f} GB/s each way (both at once)")
    del h_in, h_out, ti, to
os.sched_setaffinity(0, full)
