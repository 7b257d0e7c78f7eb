mkdir -p gpurun_out
S=gpurun_out/k5_summary.txt; : > $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/k5_mgpu4.log 2>&1; echo "mgpu4 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --no-pmg > gpurun_out/k5_bench4.json 2> gpurun_out/k5_bench4.err; echo "bench4 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --no-pmg > gpurun_out/k5_bench2.json 2> gpurun_out/k5_bench2.err; echo "bench2 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 bench.py --gpus 4 --no-pmg --ez 128 --no-beyond > gpurun_out/k5_bench4_big.json 2> gpurun_out/k5_bench4_big.err; echo "bench4big $?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-pmg --no-cpu-baseline > gpurun_out/k5_bench1.json 2> gpurun_out/k5_bench1.err; echo "bench1 $?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-pmg --ez 128 --no-beyond --no-cpu-baseline > gpurun_out/k5_bench1_big.json 2> gpurun_out/k5_bench1_big.err; echo "bench1big $?" >> $S
for f in bench4 bench2 bench4_big bench1 bench1_big; do python -c "import json;d=json.loads(open('gpurun_out/k5_$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['clocks'])" >> $S; done
