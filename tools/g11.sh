mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_multigpu.py -q -s -k "2" > gpurun_out/g11_mgpu.log 2>&1
echo "mgpu exit $?" >> gpurun_out/g11_summary.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --no-pmg > gpurun_out/g11_bench2.json 2> gpurun_out/g11_bench2.err
echo "bench2 exit $?" >> gpurun_out/g11_summary.txt
