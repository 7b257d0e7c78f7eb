mkdir -p gpurun_out
S=gpurun_out/j31_summary.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/j31_lb.log 2>&1; echo "loopback $?" >> $S
tail -1 gpurun_out/j31_lb.log >> $S
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j31_mgpu.log 2>&1; echo "mgpu $?" >> $S
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j31_b2.json 2> gpurun_out/j31_b2.err; echo "bench2 $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j31_b2.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'], d['kernel_ms_per_step'])" >> $S
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/mgpu_timeline.py --graph --iters 20 --tag _j31p2 > gpurun_out/j31_p2.log 2>&1; echo "p2 $?" >> $S
