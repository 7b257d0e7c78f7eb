"""Per-rank kernel timeline of multi-GPU PCG iterations (CUPTI through torch.profiler).

  python -m torch.distributed.run --nproc-per-node 4 --master-addr 127.0.0.1 tools/mgpu_timeline.py \
      [--mesh box|rod] [--ez 16] [--iters 20] [--graph]

Warm-up solves, then one profiled solve of --iters iterations; every rank writes
gpurun_out/timeline_r{rank}.json with the kernel records (name, stream, start/end in us relative to
the first kernel) and prints a per-iteration summary: iteration period, per-kernel-class busy time
and the gaps on the main stream (waiting for peers)."""
import argparse
import collections
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import bench  # noqa: E402
from paper_2409_19119_b200 import nek  # noqa: E402
from workloads import meshgen as mg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--mesh", default="box")
ap.add_argument("--ez", type=int, default=16)
ap.add_argument("--order", type=int, default=7)
ap.add_argument("--rod-layers", type=int, default=3)
ap.add_argument("--h2", type=float, default=0.0)
ap.add_argument("--iters", type=int, default=20)
ap.add_argument("--graph", action="store_true", help="profile the CUDA-graph path (default: eager launches)")
ap.add_argument("--tag", default="")
a = ap.parse_args()
rank, world, local = bench.rank_env()
torch.cuda.set_device(local)
dev = torch.device("cuda", local)
comm = None
if world > 1:
    dist.init_process_group("nccl", device_id=dev)
    comm = nek.comm_from_torch(dev)
if not a.graph:
    os.environ["NEK_NO_GRAPH"] = "1"
m = bench.make_mesh(rank, world, a.ez, a.order, a)
ctx = nek.setup(m.E, m.N, m.xyz, m.gid, m.mask, comm=comm, device=local)
b = torch.from_numpy(mg.smooth_field(m, seed=1)).to(dev)
x = torch.zeros_like(b)
for _ in range(3):
    nek.pcg_solve(ctx, 1.0, a.h2, b, x, 0.0, a.iters)
torch.cuda.synchronize()
if world > 1:
    dist.barrier()
from torch.profiler import ProfilerActivity, profile  # noqa: E402

with profile(activities=[ProfilerActivity.CUDA]) as prof:
    nek.pcg_solve(ctx, 1.0, a.h2, b, x, 0.0, a.iters)
    torch.cuda.synchronize()
os.makedirs("gpurun_out", exist_ok=True)
path = f"gpurun_out/trace_r{rank}.json"
prof.export_chrome_trace(path)
ev = [e for e in json.load(open(path))["traceEvents"] if e.get("cat") == "kernel"]
ev.sort(key=lambda e: e["ts"])
t0 = ev[0]["ts"] if ev else 0.0
recs = [{"name": e["name"].split("(")[0].replace("void ", "").replace("nekb200::", "").split("<")[0],
         "stream": e["args"].get("stream"), "t": round(e["ts"] - t0, 2), "d": round(e["dur"], 2)} for e in ev]
json.dump(recs, open(f"gpurun_out/timeline{a.tag}_r{rank}.json", "w"))
os.remove(path)
# per-iteration summary: iterations delimited by the update kernel on the main stream
busy = collections.defaultdict(float)
for r in recs:
    busy[r["name"]] += r["d"]
upd = [r for r in recs if r["name"].startswith("pcg_update")]
period = (upd[-1]["t"] - upd[0]["t"]) / max(1, len(upd) - 1) if len(upd) > 1 else None
out = {"rank": rank, "world": world, "E": m.E, "kernels": len(recs), "iter_period_us": period,
       "busy_us_per_iter": {k: round(v / max(1, len(upd)), 2) for k, v in sorted(busy.items(), key=lambda kv: -kv[1])},
       "first_iters": [r for r in recs if upd and len(upd) > 3 and upd[1]["t"] < r["t"] + r["d"] and r["t"] < upd[3]["t"] + 1]}
print(json.dumps(out), flush=True)
nek.free(ctx)
if world > 1:
    dist.destroy_process_group()
