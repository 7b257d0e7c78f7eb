set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 0 8; do python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline --variant $v > gpurun_out/bench9g_v$v.json 2>> gpurun_out/bench9.err; done
python bench.py --steps 10 --warmup 3 > gpurun_out/bench9.json 2>> gpurun_out/bench9.err
python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/prof_plain.log 2>&1 && ncu --set full --cache-control none --clock-control none --import-source on -k regex:"ax_v5" -s 3 -c 1 -o gpurun_out/prof_r1g python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/ncu2.log 2>&1
