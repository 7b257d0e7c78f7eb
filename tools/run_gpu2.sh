mkdir -p gpurun_out
S=gpurun_out/j29_summary.txt; : > $S
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -x -q -k "prefetch or variants or window or config2 or config3 or deferred or slab_p2p" > gpurun_out/j29_tests.log 2>&1; echo "tests $?" >> $S
tail -1 gpurun_out/j29_tests.log >> $S
timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/j29_b.json 2>gpurun_out/j29_b.err; echo "bench $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j29_b.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], 'big', d['beyond_l2']['vec_per_iter']['frac'], d['beyond_l2']['pcg_ax']['frac'], d['beyond_l2']['ax_gs']['frac'])" >> $S
