set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline --variant 10 > gpurun_out/bench14g_v10.json 2> gpurun_out/bench14.err
python bench.py --steps 5 --warmup 3 --graph --no-cpu-baseline --variant 10 --ez 128 > gpurun_out/bench14g_v10_ez128.json 2>> gpurun_out/bench14.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --mesh rod > gpurun_out/bench14_rod.json 2>> gpurun_out/bench14.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --mesh rod --h2 100 > gpurun_out/bench14_rod_vel.json 2>> gpurun_out/bench14.err
