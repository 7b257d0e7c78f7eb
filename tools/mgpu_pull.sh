# 2 GPUs: warp-parallel mailbox pulls -- bench (config 2 per GPU) and parity
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29591"
for k in 1 2; do
timeout 600 $T bench.py --gpus 2 --steps 5 --no-pmg --no-peaks > gpurun_out/pull_b2.json 2> gpurun_out/pull_b2.err
python -c "
import json; d=json.loads(open('gpurun_out/pull_b2.json').read().strip().splitlines()[-1])
print('N=2 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], d['clocks'])" || tail -5 gpurun_out/pull_b2.err
done
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
