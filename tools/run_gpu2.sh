mkdir -p gpurun_out
S=gpurun_out/j2_summary.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "deferred or window or config2 or variants or repeatable or edge or manufactured or l2_resident" > gpurun_out/j2_tests.log 2>&1; echo "tests $?" >> $S
tail -3 gpurun_out/j2_tests.log >> $S
for d in 1 0 1 0; do
  NEK_DEFER=$d timeout 300 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/j2_b$d.json 2>gpurun_out/j2_b$d.err; echo "bench defer=$d $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j2_b$d.json').read().strip().splitlines()[-1]);print('defer=$d', d['value'], d['ms_per_step'], d.get('roofline',{}).get('frac'))" >> $S
done
timeout 600 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/j2_lb.log 2>&1; echo "loopback $?" >> $S
tail -2 gpurun_out/j2_lb.log >> $S
