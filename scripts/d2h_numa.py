"""D2H bandwidth into a large pinned buffer: per 1 GB region, with the default
CPU affinity and with the process bound to the GPU's local NUMA CPUs."""
import json, os, subprocess, sys, time
import torch

def gpu_local_cpus(dev=0):
    if True:
        out = subprocess.run(["nvidia-smi", "--query-gpu=pci.bus_id", "--format=csv,noheader", "-i", str(dev)],
                             capture_output=True, text=True).stdout.strip()
        bus = out
    bus = bus.lower()
    if bus.startswith("0000") and len(bus.split(":")[0]) == 8:
        bus = bus[4:]
    path = f"/sys/bus/pci/devices/{bus}/local_cpulist"
    try:
        txt = open(path).read().strip()
    except OSError:
        return None, path
    cpus = set()
    for part in txt.split(","):
        a, _, b = part.partition("-")
        cpus.update(range(int(a), int(b or a) + 1))
    return cpus, txt

mode = sys.argv[1] if len(sys.argv) > 1 else "default"
info = {"mode": mode, "ncpu": os.cpu_count()}
cpus, txt = gpu_local_cpus()
info["gpu_local_cpulist"] = txt
if mode == "bind" and cpus:
    os.sched_setaffinity(0, cpus)
info["numa_nodes"] = subprocess.run(["bash", "-c", "ls -d /sys/devices/system/node/node* | wc -l"], capture_output=True, text=True).stdout.strip()
GB = 1 << 30
n = 16
src = torch.empty(GB // 4, dtype=torch.int32, device="cuda").fill_(1)
host = torch.empty(n * GB // 4, dtype=torch.int32, pin_memory=True)
torch.cuda.synchronize()
rates = []
for i in range(n):
    dst = host[i * GB // 4:(i + 1) * GB // 4]
    dst.copy_(src, non_blocking=True); torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(2):
        dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    rates.append(round(2 * GB / (time.perf_counter() - t0) / 1e9, 1))
info["d2h_gbs_per_region"] = rates
t0 = time.perf_counter()
hsrc = host[: GB // 4]
for _ in range(2):
    src.copy_(hsrc, non_blocking=True)
torch.cuda.synchronize()
info["h2d_gbs"] = round(2 * GB / (time.perf_counter() - t0) / 1e9, 1)
print(json.dumps(info), flush=True)
