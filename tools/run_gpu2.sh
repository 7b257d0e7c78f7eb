mkdir -p gpurun_out
S=gpurun_out/j12_summary.txt; : > $S
for pf in 1 0 1 0; do
  NEK_GS_PFL1=$pf timeout 300 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/j12_b.json 2>gpurun_out/j12_b.err; echo "bench pf=$pf $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j12_b.json').read().strip().splitlines()[-1]);print('pf=$pf', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['gs_ms'], 'axgs', d['ax_gs']['gs_kernel']['avg_launch_ms'], d['ax_gs']['gs_kernel']['frac'], 'big', d['beyond_l2']['gs']['avg_launch_ms'], d['beyond_l2']['gs']['frac'], d['beyond_l2']['ax_gs']['frac'])" >> $S
done
