# Ax v5 configurations at config 2 with the L2-resident vectors: 0 (auto: TMA metric ring, 3 CTAs/SM),
# 8 (registers, 3/SM), 9 (registers + bulk L2 prefetch of the next element, 4/SM)
for v in 0 8 9 0; do
  timeout 300 python bench.py --steps 5 --warmup 3 --no-pmg --no-peaks --no-cpu-baseline --variant $v > gpurun_out/var_$v.json 2> gpurun_out/var_$v.err
  python -c "
import json; d=json.loads(open('gpurun_out/var_$v.json').read().strip().splitlines()[-1])
print('variant $v', 'GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), {k: round(x,3) for k,x in d['kernel_ms_per_step'].items()}, 'frac %.3f' % d['roofline']['frac'])" || tail -3 gpurun_out/var_$v.err
done
