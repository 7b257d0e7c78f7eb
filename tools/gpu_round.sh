set -x
NEK_DEBUG=1 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench13.json 2> gpurun_out/bench13.err
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
timeout 600 python tools/nsweep.py > gpurun_out/nsweep.jsonl 2> gpurun_out/nsweep.err
