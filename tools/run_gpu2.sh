mkdir -p gpurun_out
S=gpurun_out/j40_summary.txt; : > $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q -k "deferred or window or config2 or edge or manufactured or prefetch or repeatable or l2_resident or slab_p2p" > gpurun_out/j40_t.log 2>&1; echo "tests $?" >> $S
tail -1 gpurun_out/j40_t.log >> $S
for i in 1 2; do
  timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/j40_b.json 2>gpurun_out/j40_b.err; echo "bench $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j40_b.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['kernel_ms_per_step']['vec_ms'], 'big', d['beyond_l2']['vec_per_iter']['frac'], d['gpu_launches'])" >> $S
done
