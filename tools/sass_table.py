"""SASS evidence table for profiles/r2_sass.md: per kernel instantiation of libnek.so, the counts of
DMMA (FP64 tensor-core mma), UBLKCP (cp.async.bulk TMA copies), UBLKPF (cp.async.bulk.prefetch.L2),
SYNCS (mbarrier ops), DFMA, plus registers and stack from cuobjdump -res-usage.

  python tools/sass_table.py [libnek.so] > profiles/r2_sass.md
"""
import collections
import re
import subprocess
import sys

lib = sys.argv[1] if len(sys.argv) > 1 else "paper_2409_19119_b200/libnek.so"
KEEP = ("ax_v5_kernel", "ax_v6_kernelILi8", "gs_chunk_kernel", "gs_classes_kernel", "pcg_update_deferred",
        "pcg_update_fused", "makef_mma_kernel", "gs_classes_unpack_kernel", "gs_pack_p2p_fused")
sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
res = subprocess.run(["cuobjdump", "-res-usage", lib], capture_output=True, text=True).stdout
usage = {}
for fn, line in re.findall(r"Function (\S+):\n\s*(REG:.*)", res):
    reg = re.search(r"REG:(\d+)", line).group(1)
    stk = re.search(r"STACK:(\d+)", line).group(1)
    usage[fn] = (reg, stk)
counts = collections.OrderedDict()
cur = None
for ln in sass.splitlines():
    m = re.search(r"Function : (\S+)", ln)
    if m:
        cur = m.group(1) if any(k in m.group(1) for k in KEEP) else None
        if cur:
            counts[cur] = collections.Counter()
        continue
    if cur:
        for op in ("DMMA", "UBLKCP", "UBLKPF", "SYNCS", "DFMA"):
            if re.search(r"\b" + op, ln):
                counts[cur][op] += 1
print("# SASS evidence (cuobjdump -sass paper_2409_19119_b200/libnek.so, final round-2 code)\n")
print("Instruction counts per kernel instantiation (`tools/sass_table.py`): DMMA = FP64 tensor-core "
      "mma.sync.m8n8k4 (Ax v5 r/s contractions, makef stages), UBLKCP = cp.async.bulk (TMA bulk copies into "
      "shared memory), UBLKPF = cp.async.bulk.prefetch.L2 (bulk L2 prefetch: large-launch v5 Ax, residual "
      "update), SYNCS = mbarrier operations, DFMA = FP64 FMA; registers and stack bytes from "
      "cuobjdump -res-usage.  tcgen05 has no FP64 kind, so UTC*MMA / TMEM do not apply to this FP64 path.\n")
print("| kernel (mangled) | DMMA | UBLKCP | UBLKPF | SYNCS | DFMA | regs | stack |")
print("|---|---|---|---|---|---|---|---|")
for fn, c in sorted(counts.items()):
    reg, stk = usage.get(fn, ("?", "?"))
    print(f"| `{fn[:110]}` | {c['DMMA']} | {c['UBLKCP']} | {c['UBLKPF']} | {c['SYNCS']} | {c['DFMA']} | {reg} | {stk} |")
