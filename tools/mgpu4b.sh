# 4 GPUs: default bench (config 2 per GPU, all sections) -- the driver's scaling command
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561"
timeout 900 $T bench.py --gpus 4 --steps 5 > gpurun_out/g4b_bench.json 2> gpurun_out/g4b_bench.err; echo rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/g4b_bench.json').read().strip().splitlines()[-1])
print('GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], d['halo'], d['clocks'], d['pmg']['ms'], d['pmg']['iters'], d['projection']['iters_L8'], d['peaks_box'].get('nccl_allreduce_latency'), d['peaks_box'].get('nccl_sendrecv_GBps_rank0_to_1'))" || tail -20 gpurun_out/g4b_bench.err
