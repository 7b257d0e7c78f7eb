# 2 GPUs: per-slot gather list in the P2P halo pack -- bench, parity, timeline
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611"
for k in 1 2; do
timeout 600 $T bench.py --gpus 2 --steps 5 --no-pmg --no-peaks > gpurun_out/pack_b2.json 2> gpurun_out/pack_b2.err
python -c "
import json; d=json.loads(open('gpurun_out/pack_b2.json').read().strip().splitlines()[-1])
print('N=2 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'])" || tail -5 gpurun_out/pack_b2.err
done
timeout 600 $T tools/mgpu_check.py > gpurun_out/pack_check.log 2>&1; grep '^{' gpurun_out/pack_check.log | tail -1 | cut -c1-120; echo
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
timeout 600 $T bench.py --gpus 2 --steps 3 --mesh rod --no-pmg --no-peaks > gpurun_out/pack_rod.json 2> gpurun_out/pack_rod.err
python -c "
import json; d=json.loads(open('gpurun_out/pack_rod.json').read().strip().splitlines()[-1])
print('rod N=2 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], d['halo']['GBps'])" || tail -5 gpurun_out/pack_rod.err
