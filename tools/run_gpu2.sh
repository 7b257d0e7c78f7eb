mkdir -p gpurun_out
S=gpurun_out/j42_summary.txt; : > $S
for v in 0 8 0 8; do
  timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-pmg --variant $v > gpurun_out/j42_b.json 2>gpurun_out/j42_b.err; echo "bench v=$v $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j42_b.json').read().strip().splitlines()[-1]);print('v=$v', d['value'], 'axgs', d['ax_gs']['frac'], 'big', d['beyond_l2']['ax_gs']['frac'], d['beyond_l2']['pcg_ax']['frac'])" >> $S
done
