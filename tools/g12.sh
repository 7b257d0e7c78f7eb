mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pmg.py -q -s > gpurun_out/g12_pmg.log 2>&1
echo "pmg exit $?" >> gpurun_out/g12_summary.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "window or config2_full or variants" > gpurun_out/g12_par.log 2>&1
echo "par exit $?" >> gpurun_out/g12_summary.txt
timeout 400 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/g12_bench.json 2> gpurun_out/g12_bench.err
echo "bench exit $?" >> gpurun_out/g12_summary.txt
