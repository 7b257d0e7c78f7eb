# 2 GPUs: config-2-per-GPU weak scaling bench, CUPTI timeline of the graph path, multi-GPU parity
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511"
timeout 400 $T bench.py --gpus 2 --steps 5 --warmup 3 --no-pmg > gpurun_out/m2_bench.json 2> gpurun_out/m2_bench.err; tail -c 2500 gpurun_out/m2_bench.json
timeout 300 $T tools/mgpu_timeline.py --graph --iters 20 > gpurun_out/m2_tl.log 2>&1; tail -c 6000 gpurun_out/m2_tl.log
timeout 600 python -m pytest tests/test_multigpu.py -x -q > gpurun_out/m2_pytest.log 2>&1; tail -3 gpurun_out/m2_pytest.log
