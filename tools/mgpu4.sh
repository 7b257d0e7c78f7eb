# 4 GPUs: default bench (config 2 per GPU, weak), rod bundle (config 4, weak), config 3 (strong), parity
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541"
s() { python -c "
import json,sys; d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], 'GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], 'halo', d['halo'].get('GBps'), d['clocks'], 'pmg', (d.get('pmg') or {}).get('ms'), (d.get('pmg') or {}).get('iters'), 'peaks', (d.get('peaks_box') or {}).get('nccl_allreduce_latency'), (d.get('peaks_box') or {}).get('nccl_sendrecv_GBps_rank0_to_1'))" "$1" || tail -5 "${1%.json}.err"; }
timeout 900 $T bench.py --gpus 4 > gpurun_out/g4_bench.json 2> gpurun_out/g4_bench.err; s gpurun_out/g4_bench.json
timeout 900 $T bench.py --gpus 4 --mesh rod --no-pmg --no-peaks --steps 3 > gpurun_out/g4_rod.json 2> gpurun_out/g4_rod.err; s gpurun_out/g4_rod.json
timeout 900 $T bench.py --gpus 4 --mesh cfg3 --no-pmg --no-peaks --steps 3 > gpurun_out/g4_cfg3.json 2> gpurun_out/g4_cfg3.err; s gpurun_out/g4_cfg3.json
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
