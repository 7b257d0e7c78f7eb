mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py -q -s > gpurun_out/g3_par.log 2>&1
echo "par exit $?" >> gpurun_out/g3_summary.txt
timeout 900 python bench.py > gpurun_out/g3_bench.json 2> gpurun_out/g3_bench.err
echo "bench exit $?" >> gpurun_out/g3_summary.txt
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/g3_ref.json 2> gpurun_out/g3_ref.err
echo "ref exit $?" >> gpurun_out/g3_summary.txt
