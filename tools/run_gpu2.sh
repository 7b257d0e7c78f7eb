mkdir -p gpurun_out
S=gpurun_out/j38_summary.txt; : > $S
NEK_BND_ONE=1 NEK_P2P_TIMEOUT_MS=5000 timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j38_mgpu.log 2>&1; echo "mgpu one $?" >> $S
grep -o '"ok": [a-z]*' gpurun_out/j38_mgpu.log | head -3 >> $S
for o in 1 0 1 0; do
NEK_BND_ONE=$o NEK_P2P_TIMEOUT_MS=5000 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j38_b2.json 2> gpurun_out/j38_b2.err; echo "bench2 one=$o $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j38_b2.json').read().strip().splitlines()[-1]);print('one=$o', d['value'], d['ms_per_step'])" >> $S
done
NEK_BND_ONE=1 timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 tools/mgpu_timeline.py --graph --iters 20 --tag _j38p2 > gpurun_out/j38_p2.log 2>&1; echo "p2 $?" >> $S
