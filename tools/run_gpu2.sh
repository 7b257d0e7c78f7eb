mkdir -p gpurun_out
S=gpurun_out/j34_summary.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_loopback.py -x -q > gpurun_out/j34_lb.log 2>&1; echo "loopback $?" >> $S
tail -1 gpurun_out/j34_lb.log >> $S
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j34_mgpu4.log 2>&1; echo "mgpu4 $?" >> $S
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j34_b4.json 2> gpurun_out/j34_b4.err; echo "bench4 $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j34_b4.json').read().strip().splitlines()[-1]);print('4', d['value'], d['ms_per_step'])" >> $S
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j34_b2.json 2> gpurun_out/j34_b2.err; echo "bench2 $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j34_b2.json').read().strip().splitlines()[-1]);print('2', d['value'], d['ms_per_step'])" >> $S
done
