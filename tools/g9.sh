mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "xlink or window or config2 or variants or ax_parity or gs_values or repeatable or rod" > gpurun_out/g9_par.log 2>&1
echo "par exit $?" >> gpurun_out/g9_summary.txt
timeout 400 python bench.py --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g9_bench.json 2> gpurun_out/g9_bench.err
echo "bench exit $?" >> gpurun_out/g9_summary.txt
NEK_XLINK=0 timeout 400 python bench.py --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g9_bench0.json 2> gpurun_out/g9_bench0.err
echo "bench0 exit $?" >> gpurun_out/g9_summary.txt
