# 2 GPUs: concurrent boundary/interior Ax sharing one wave (NEK_BND_SPLIT) -- A/B and parity
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29601"
for sp in 1 0 1 0; do
NEK_BND_SPLIT=$sp timeout 600 $T bench.py --gpus 2 --steps 5 --no-pmg --no-peaks > gpurun_out/split_$sp.json 2> gpurun_out/split_$sp.err
python -c "
import json; d=json.loads(open('gpurun_out/split_$sp.json').read().strip().splitlines()[-1])
print('split=$sp N=2 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/split_$sp.err
done
timeout 600 $T tools/mgpu_check.py > gpurun_out/split_check.log 2>&1; grep '^{' gpurun_out/split_check.log | tail -1 | cut -c1-150; echo
timeout 300 $T tools/mgpu_timeline.py --graph --iters 20 > gpurun_out/split_tl.log 2>&1; grep '^{' gpurun_out/split_tl.log | cut -c1-700
