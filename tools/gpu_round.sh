timeout 600 python -m pytest tests/test_gpu_pmg.py -x -q > gpurun_out/pytest_pmg.log 2>&1; tail -30 gpurun_out/pytest_pmg.log
timeout 300 python tools/pmg_bench.py --ez 16 > gpurun_out/pmgb_ez16.jsonl 2>&1; cat gpurun_out/pmgb_ez16.jsonl
timeout 300 python tools/pmg_bench.py --ez 16 --coarse-degree 40 --coarse-lo 0.5 > gpurun_out/pmgb_ez16b.jsonl 2>&1; cat gpurun_out/pmgb_ez16b.jsonl
echo done
