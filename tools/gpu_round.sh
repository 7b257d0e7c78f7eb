timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k config3 > gpurun_out/pytest_cfg3.log 2>&1; tail -3 gpurun_out/pytest_cfg3.log
