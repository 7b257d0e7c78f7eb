mkdir -p gpurun_out
for c in 2 4 8; do NEK_UPD_CTAS=$c timeout 300 python bench.py --no-beyond --no-cpu-baseline --no-peaks --no-pmg > gpurun_out/g6_upd$c.json 2> gpurun_out/g6_upd$c.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "window or config2_full or variants" > gpurun_out/g6_par.log 2>&1
echo "par exit $?" >> gpurun_out/g6_summary.txt
