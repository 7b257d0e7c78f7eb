# A/B: programmatic dependent launch on the per-iteration kernels, config 2; parity tests
run() {  # tag, env...
  tag=$1; shift
  env "$@" timeout 300 python bench.py --steps 5 --warmup 3 --no-pmg --no-peaks --no-cpu-baseline > gpurun_out/ab_$tag.json 2> gpurun_out/ab_$tag.err
  python - "$tag" <<'PY'
import json, sys
try:
    d = json.loads(open(f"gpurun_out/ab_{sys.argv[1]}.json").read().strip().splitlines()[-1])
    print(sys.argv[1], "GDOF/s %.2f iter/s %.0f" % (d["value"], d["pcg_iter_per_s"]),
          "kernel_ms", {k: round(v, 3) for k, v in d["kernel_ms_per_step"].items()}, "ax frac %.3f" % d["roofline"]["frac"],
          "axgs %.2f" % d["ax_gs"]["gdof_per_s"], "e2e %.2f" % d["e2e"]["value"], "clk", d["clocks"]["sm_mhz"], flush=True)
except Exception as e:
    print(sys.argv[1], "FAILED", e, open(f"gpurun_out/ab_{sys.argv[1]}.err").read()[-1500:], flush=True)
PY
}
run pdl0 NEK_PDL=0
run pdl1 NEK_PDL=1
run pdl1b NEK_PDL=1
run pdl0b NEK_PDL=0
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_pmg.py tests/test_gpu_makef.py -x -q 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
