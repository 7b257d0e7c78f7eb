mkdir -p gpurun_out
S=gpurun_out/k7_summary.txt; : > $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/k7_mgpu4.log 2>&1; echo "mgpu4 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 4 --no-pmg > gpurun_out/k7_bench4.json 2> gpurun_out/k7_bench4.err; echo "bench4 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29633 bench.py --gpus 2 --no-pmg > gpurun_out/k7_bench2.json 2> gpurun_out/k7_bench2.err; echo "bench2 $?" >> $S
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29634 bench.py --gpus 4 --no-pmg --ez 128 --no-beyond > gpurun_out/k7_bench4_big.json 2> gpurun_out/k7_bench4_big.err; echo "bench4big $?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --no-pmg --no-cpu-baseline --no-beyond > gpurun_out/k7_bench1.json 2> gpurun_out/k7_bench1.err; echo "bench1 $?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --mesh cfg3 --steps 3 --warmup 3 --no-pmg --no-cpu-baseline --no-beyond > gpurun_out/k7_cfg3.json 2> gpurun_out/k7_cfg3.err; echo "cfg3 $?" >> $S
CUDA_VISIBLE_DEVICES=0 timeout 900 python bench.py --mesh rod --steps 5 --warmup 3 --no-pmg --no-cpu-baseline --no-beyond > gpurun_out/k7_rod.json 2> gpurun_out/k7_rod.err; echo "rod $?" >> $S
for f in bench4 bench2 bench4_big bench1 cfg3 rod; do python -c "import json;d=json.loads(open('gpurun_out/k7_$f.json').read().strip().splitlines()[-1]);print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['ax_gs']['frac'], d['clocks'])" >> $S; done
