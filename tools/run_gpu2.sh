mkdir -p gpurun_out
R="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -x > gpurun_out/g4_loop.log 2>&1; echo "loop $?" >> gpurun_out/g4_summary.txt
timeout 600 $R --nproc-per-node 4 --master-port 29662 bench.py --gpus 4 --no-pmg --no-peaks > gpurun_out/g4_bench4.json 2> gpurun_out/g4_bench4.err; echo "bench4 $?" >> gpurun_out/g4_summary.txt
timeout 600 $R --nproc-per-node 2 --master-port 29664 bench.py --gpus 2 --no-pmg --no-peaks > gpurun_out/g4_bench2.json 2> gpurun_out/g4_bench2.err; echo "bench2 $?" >> gpurun_out/g4_summary.txt
timeout 600 $R --nproc-per-node 4 --master-port 29665 tools/mgpu_timeline.py --graph --iters 20 > gpurun_out/g4_timeline.log 2>&1; echo "timeline $?" >> gpurun_out/g4_summary.txt
