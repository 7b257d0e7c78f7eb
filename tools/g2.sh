mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -s -k "window or config2 or rod or variants or generic or loopback_slab_p2p or block or staged" > gpurun_out/g2_par.log 2>&1
echo "par exit $?" >> gpurun_out/g2_summary.txt
timeout 600 python bench.py > gpurun_out/g2_bench.json 2> gpurun_out/g2_bench.err
echo "bench exit $?" >> gpurun_out/g2_summary.txt
