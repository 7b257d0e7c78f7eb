# 1 GPU full bench, PCG parity subset, 2-GPU default bench and multi-GPU parity
CUDA_VISIBLE_DEVICES=0 timeout 600 python bench.py > gpurun_out/r3_b1.json 2> gpurun_out/r3_b1.err
python -c "
import json; d=json.loads(open('gpurun_out/r3_b1.json').read().strip().splitlines()[-1])
print('N=1 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], 'frac %.3f' % d['roofline']['frac'], 'axgs %.2f' % d['ax_gs']['gdof_per_s'], 'e2e %.2f' % d['e2e']['value'], d['clocks'], 'pmg', d['pmg']['ms'], d['pmg']['fp32']['ms'], 'makef', d['makef']['ms_per_apply'], d['cpu_baseline'])" || tail -5 gpurun_out/r3_b1.err
CUDA_VISIBLE_DEVICES=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29581"
timeout 600 $T bench.py --gpus 2 --steps 5 > gpurun_out/r3_b2.json 2> gpurun_out/r3_b2.err
python -c "
import json; d=json.loads(open('gpurun_out/r3_b2.json').read().strip().splitlines()[-1])
print('N=2 GDOF/s %.2f iter/s %.0f' % (d['value'], d['pcg_iter_per_s']), d['kernel_ms_per_step'], d['clocks'], d['peaks_box'].get('nccl_sendrecv_GBps_rank0_to_1'))" || tail -5 gpurun_out/r3_b2.err
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
