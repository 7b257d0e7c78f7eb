# Config-2 PCG tuning sweep: L2-resident vectors (NEK_L2KEEP / set-aside), gs pairs per
# thread (NEK_GS_PPT), residual-update CTAs per SM (NEK_UPD_CFG)
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-pmg --no-peaks --no-cpu-baseline > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err
  python - "$tag" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/sw_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "GDOF/s %.2f iter/s %.0f" % (d["value"], d["pcg_iter_per_s"]),
          "kernel_ms", {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, "ax frac %.3f" % d["roofline"]["frac"],
          "axgs %.2f" % d["ax_gs"]["gdof_per_s"], "clk", d["clocks"]["sm_mhz"], flush=True)
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(f"gpurun_out/sw_{sys.argv[1]}.err").read()[-800:], flush=True)
PY
}
run k0 NEK_L2KEEP=0
run k1 NEK_L2KEEP=1
run k3 NEK_L2KEEP=3
run k0sa NEK_L2KEEP=0 NEK_L2SETASIDE=96
run k1sa NEK_L2KEEP=1 NEK_L2SETASIDE=96
run k3sa NEK_L2KEEP=3 NEK_L2SETASIDE=96
for p in 1 2 4; do run ppt$p NEK_GS_PPT=$p; done
for u in 4 8; do run upd$u NEK_UPD_CFG=$u; done
timeout 300 python -c "
from paper_2409_19119_b200 import nek
print('hbm', nek.probe_hbm_gbps(0), 'smem', nek.probe_smem_tbps(0), 'dfma', nek.probe_fp64_tflops(0))"
NEK_L2KEEP=3 NEK_GS_PPT=2 NEK_UPD_CFG=4 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
