mkdir -p gpurun_out
S=gpurun_out/j27_summary.txt; : > $S
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "gs" > gpurun_out/j27_tests.log 2>&1; echo "tests $?" >> $S
tail -1 gpurun_out/j27_tests.log >> $S
for pf in 1 0 1 0; do
  NEK_GS_PF=$pf timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/j27_b.json 2>gpurun_out/j27_b.err; echo "bench pf=$pf $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j27_b.json').read().strip().splitlines()[-1]);print('pf=$pf', d['value'], d['ms_per_step'], d['ax_gs']['gs_kernel']['avg_launch_ms'], 'big', d['beyond_l2']['gs']['avg_launch_ms'], d['beyond_l2']['gs']['frac'], d['beyond_l2']['ax_gs']['frac'])" >> $S
done
