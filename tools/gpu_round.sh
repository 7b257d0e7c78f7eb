set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 0 5 4 3 2 1; do python tools/prof_step.py --variant $v --solves 0 --ax 30 > gpurun_out/var_$v.log 2>&1; done
for v in 0 5 4; do python tools/prof_step.py --variant $v --solves 0 --ax 30 --h2 1.0 > gpurun_out/varh_$v.log 2>&1; done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench4.json 2> gpurun_out/bench4.err
python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline > gpurun_out/bench4g.json 2>> gpurun_out/bench4.err
python tools/prof_step.py > gpurun_out/prof_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:"ax_v3|gs_classes" -s 4 -c 2 -o gpurun_out/prof_r1c python tools/prof_step.py > gpurun_out/ncu2.log 2>&1
