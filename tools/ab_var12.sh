# config 2: default (register streaming at 3 CTAs/SM for the fused L2-resident launch) vs variant 12 (4 CTAs/SM)
for v in 0 12 0 12; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-pmg --no-peaks --no-cpu-baseline --variant $v > gpurun_out/v12_$v.json 2> gpurun_out/v12_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/v12_$v.json').read().strip().splitlines()[-1])
print('variant $v', 'GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()}, 'frac %.3f' % d['roofline']['frac'], 'axgs %.2f' % d['ax_gs']['gdof_per_s'])" || tail -3 gpurun_out/v12_$v.err
done
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "variants_N7" 2>&1 | tail -2
