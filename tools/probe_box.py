"""One-off probe of the GPU box: host RAM, cores, PCIe H2D/D2H bandwidth."""
import os, subprocess, time, json
import torch
out = {}
out["nproc"] = os.cpu_count()
out["affinity"] = len(os.sched_getaffinity(0))
with open("/proc/meminfo") as f:
    for line in f:
        if line.startswith(("MemTotal", "MemAvailable", "HugePages_Total")):
            k, v = line.split(":"); out[k] = v.strip()
out["smi"] = subprocess.run(["nvidia-smi", "--query-gpu=name,pci.bus_id,pcie.link.gen.max,pcie.link.width.max,memory.total,clocks.max.sm", "--format=csv"], capture_output=True, text=True).stdout
out["topo"] = subprocess.run(["nvidia-smi", "topo", "-m"], capture_output=True, text=True).stdout
dev = torch.device("cuda:0")
for gib in (1,):
    n = gib << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        best = 0
        for _ in range(6):
            s = torch.cuda.Event(enable_timing=True); e = torch.cuda.Event(enable_timing=True)
            s.record(); fn(); e.record(); torch.cuda.synchronize()
            best = max(best, n / (s.elapsed_time(e) * 1e-3) / 1e9)
        out[f"{name}_gbs_{gib}g"] = best
    # bidirectional
    s2 = torch.cuda.Stream()
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True); d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    out["bidir_gbs_total"] = 2 * n / dt / 1e9
t = time.perf_counter()
big = torch.empty(32 << 30, dtype=torch.uint8, pin_memory=True)
out["pin_32g_s"] = time.perf_counter() - t
print(json.dumps(out, indent=1))
