# 2 GPUs: folded P2P bookkeeping -- parity (both Ax orderings) and config-2-per-GPU bench A/B
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py --steps 5 --no-cpu-baseline > gpurun_out/fold_b1gpu.json 2> gpurun_out/fold_b1gpu.err; python -c "
import json; d=json.loads(open('gpurun_out/fold_b1gpu.json').read().strip().splitlines()[-1])
print('1gpu', d['value'], d['pcg_iter_per_s'], d['ax_gs'], d['pmg']['ms'], d['pmg']['ms_per_vcycle'], d['peaks_box']['hbm_fp64_GBps'], d['makef']['ms_per_apply'])" || tail -3 gpurun_out/fold_b1gpu.err
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29521"
timeout 600 $T tools/mgpu_check.py > gpurun_out/fold_check.log 2>&1; grep '^{' gpurun_out/fold_check.log | tail -1 | cut -c1-600; echo
NEK_CONCURRENT_BND=0 timeout 600 $T tools/mgpu_check.py > gpurun_out/fold_check_so.log 2>&1; grep '^{' gpurun_out/fold_check_so.log | tail -1 | cut -c1-300; echo
for f in 0 1; do
  NEK_FOLD=$f timeout 400 $T bench.py --gpus 2 --steps 5 --warmup 3 --no-pmg --no-peaks > gpurun_out/fold_b$f.json 2> gpurun_out/fold_b$f.err
  python -c "
import json; d=json.loads(open('gpurun_out/fold_b$f.json').read().strip().splitlines()[-1])
print('fold $f', 'GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], d['halo'].get('GBps'))" || tail -5 gpurun_out/fold_b$f.err
done
NEK_FOLD=1 timeout 400 $T bench.py --gpus 2 --steps 3 --warmup 3 --no-pmg --no-peaks --mesh rod > gpurun_out/fold_rod.json 2> gpurun_out/fold_rod.err; tail -c 400 gpurun_out/fold_rod.json
