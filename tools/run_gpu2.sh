mkdir -p gpurun_out
S=gpurun_out/j41_summary.txt; : > $S
NEK_UPD_CTAS=3 timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j41_mgpu.log 2>&1; echo "mgpu $?" >> $S
for c in 3 2 3 2; do
NEK_UPD_CTAS=$c timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j41_b2.json 2> gpurun_out/j41_b2.err; echo "bench2 c=$c $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j41_b2.json').read().strip().splitlines()[-1]);print('c=$c', d['value'], d['ms_per_step'])" >> $S
done
