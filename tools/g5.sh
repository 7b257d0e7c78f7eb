mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -q -s -x -k "fold or window or config2_full or variants or generic" > gpurun_out/g5_par.log 2>&1
echo "par exit $?" >> gpurun_out/g5_summary.txt
timeout 600 python bench.py --no-beyond --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g5_bench.json 2> gpurun_out/g5_bench.err
echo "bench exit $?" >> gpurun_out/g5_summary.txt
NEK_GS_FOLD=0 timeout 600 python bench.py --no-beyond --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g5_bench_nofold.json 2> gpurun_out/g5_bench_nofold.err
echo "bench0 exit $?" >> gpurun_out/g5_summary.txt
