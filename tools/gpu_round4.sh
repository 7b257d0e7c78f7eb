CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 5 --no-pmg --no-peaks --no-cpu-baseline > gpurun_out/r4_b1.json 2> gpurun_out/r4_b1.err
python -c "
import json; d=json.loads(open('gpurun_out/r4_b1.json').read().strip().splitlines()[-1])
print('N=1 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'axgs %.2f' % d['ax_gs']['gdof_per_s'], d['clocks'])" || tail -5 gpurun_out/r4_b1.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
bash tools/mgpu_pull.sh
