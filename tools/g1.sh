mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 900 python -m pytest tests/test_gpu_loopback.py -q -s -x -k "slab_p2p and 2" > gpurun_out/g1_loop_quick.log 2>&1
echo "quick exit $?" >> gpurun_out/g1_summary.txt
timeout 1500 python -m pytest tests -m gpu -q -s > gpurun_out/g1_gpu.log 2>&1
echo "gpu exit $?" >> gpurun_out/g1_summary.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/g1_summary.txt
timeout 600 python bench.py > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err
echo "bench exit $?" >> gpurun_out/g1_summary.txt
