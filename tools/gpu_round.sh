set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench15.json 2> gpurun_out/bench15.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ez 128 > gpurun_out/bench15_ez128.json 2>> gpurun_out/bench15.err
timeout 900 python tools/nsweep.py 3 4 5 6 8 9 > gpurun_out/nsweep.jsonl 2> gpurun_out/nsweep.err
