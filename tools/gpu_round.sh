timeout 900 python -m pytest tests/test_gpu_makef.py -x -q > gpurun_out/pytest_makef.log 2>&1; tail -3 gpurun_out/pytest_makef.log
for v in 0 1 2; do NEK_MAKEF_VARIANT=$v timeout 300 python tools/makef_bench.py > gpurun_out/makef_v$v.json 2>&1; echo "v$v"; cat gpurun_out/makef_v$v.json; done
for n in 3 5; do timeout 300 python tools/makef_bench.py --order $n > gpurun_out/makef_n$n.json 2>&1; cat gpurun_out/makef_n$n.json; done
echo done
