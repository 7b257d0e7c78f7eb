"""Probe the B200 box: device attributes, host cores, FP64 stream bandwidth (torch copy), clocks."""
import os, json, subprocess, time
import torch
p = torch.cuda.get_device_properties(0)
out = {"name": p.name, "sms": p.multi_processor_count, "total_mem": p.total_memory,
       "L2": getattr(p, "L2_cache_size", None), "cc": [p.major, p.minor],
       "host_cores_affinity": len(os.sched_getaffinity(0)), "cpu_count": os.cpu_count()}
try:
    out["lscpu"] = subprocess.run(["lscpu"], capture_output=True, text=True).stdout.splitlines()[:16]
except Exception as e:
    out["lscpu"] = str(e)
n = 1 << 28  # 2 GiB fp64
a = torch.randn(n, dtype=torch.float64, device="cuda"); b = torch.empty_like(a)
for _ in range(3): b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(True), torch.cuda.Event(True)
    s.record(); b.copy_(a); e.record(); e.synchronize()
    best = min(best, s.elapsed_time(e))
out["fp64_copy_GBps"] = 2 * n * 8 / best / 1e6
print(json.dumps(out, indent=1))
