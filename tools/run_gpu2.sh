mkdir -p gpurun_out
S=gpurun_out/j16_summary.txt; : > $S
true
tail -1 gpurun_out/j16_tests.log >> $S
for g in 1 1; do
  NEK_GSUPD=$g timeout 300 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/j16_b.json 2>gpurun_out/j16_b.err; echo "bench gsupd=$g $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j16_b.json').read().strip().splitlines()[-1]);print('gsupd=$g', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['beyond_l2']['vec_per_iter']['ms'], d['beyond_l2']['pcg_ax']['frac'])" >> $S
done
