mkdir -p gpurun_out
S=gpurun_out/j32_summary.txt; : > $S
timeout 900 python -m pytest tests/test_gpu_loopback.py tests/test_gpu_parity.py -x -q -k "loopback or deferred or window or config2 or edge or manufactured" > gpurun_out/j32_t.log 2>&1; echo "tests $?" >> $S
tail -1 gpurun_out/j32_t.log >> $S
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j32_mgpu.log 2>&1; echo "mgpu $?" >> $S
for i in 1 2; do
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus 2 --no-pmg --no-cpu-baseline --no-peaks --no-beyond > gpurun_out/j32_b2.json 2> gpurun_out/j32_b2.err; echo "bench2 $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j32_b2.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'])" >> $S
done
CUDA_VISIBLE_DEVICES=0 timeout 300 python bench.py --no-cpu-baseline --no-peaks --no-pmg --no-beyond > gpurun_out/j32_b1.json 2>gpurun_out/j32_b1.err; echo "bench1 $?" >> $S
python -c "import json;d=json.loads(open('gpurun_out/j32_b1.json').read().strip().splitlines()[-1]);print(d['value'], d['ms_per_step'])" >> $S
