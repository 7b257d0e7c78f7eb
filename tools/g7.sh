mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "window or config2 or variants or repeatable or edge or manufactured or l2_resident or projection" > gpurun_out/g7_par.log 2>&1
echo "par exit $?" >> gpurun_out/g7_summary.txt
timeout 300 python bench.py --no-beyond --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g7_bench.json 2> gpurun_out/g7_bench.err
echo "bench exit $?" >> gpurun_out/g7_summary.txt
NEK_PCG3=0 timeout 300 python bench.py --no-beyond --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g7_bench0.json 2> gpurun_out/g7_bench0.err
echo "bench0 exit $?" >> gpurun_out/g7_summary.txt
