mkdir -p gpurun_out
S=gpurun_out/j3_summary.txt; : > $S
NEK_PDL=1 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deferred or window or config2 or variants or repeatable or edge or manufactured or l2_resident" > gpurun_out/j3_tests.log 2>&1; echo "tests pdl $?" >> $S
tail -3 gpurun_out/j3_tests.log >> $S
for d in 1 0 1 0 1; do
  NEK_PDL=$d timeout 300 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/j3_b$d.json 2>gpurun_out/j3_b$d.err; echo "bench pdl=$d $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j3_b$d.json').read().strip().splitlines()[-1]);print('pdl=$d', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'), d['kernel_ms_per_step'])" >> $S
done
