# Config-2 PCG: L2-resident vectors (NEK_L2KEEP, persisting set-aside NEK_L2SETASIDE in MiB)
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-pmg --no-peaks --no-cpu-baseline > gpurun_out/sw_$tag.json 2> gpurun_out/sw_$tag.err
  python - "$tag" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/sw_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "GDOF/s %.2f iter/s %.0f" % (d["value"], d["pcg_iter_per_s"]),
          "kernel_ms", {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, "ax frac %.3f" % d["roofline"]["frac"],
          "axgs %.2f" % d["ax_gs"]["gdof_per_s"], "clk", d["clocks"]["sm_mhz"], d["config"]["l2_resident"], flush=True)
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(f"gpurun_out/sw_{sys.argv[1]}.err").read()[-800:], flush=True)
PY
}
run k0 NEK_L2KEEP=0
run k1 NEK_L2KEEP=1
run k3 NEK_L2KEEP=3
run k1s40 NEK_L2KEEP=1 NEK_L2SETASIDE=40
run k3s120 NEK_L2KEEP=3 NEK_L2SETASIDE=120
run auto
