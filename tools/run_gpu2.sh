mkdir -p gpurun_out
S=gpurun_out/j22_summary.txt; : > $S
for w in 2 0 1 3 4 2 0; do
  NEK_PF_WAVES=$w timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-beyond --no-pmg > gpurun_out/j22_b.json 2>gpurun_out/j22_b.err; echo "bench w=$w $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j22_b.json').read().strip().splitlines()[-1]);print('w=$w', d['value'], d['ms_per_step'], d['kernel_ms_per_step'], d['roofline']['frac'])" >> $S
done
