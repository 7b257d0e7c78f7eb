set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
for v in 0 7 3; do python tools/prof_step.py --variant $v --solves 0 --ax 30 --flush > gpurun_out/var_$v.log 2>&1; done
for v in 0 7; do python tools/prof_step.py --variant $v --solves 0 --ax 30 --h2 1.0 --flush > gpurun_out/varh_$v.log 2>&1; done
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench6.json 2> gpurun_out/bench6.err
python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline > gpurun_out/bench6g.json 2>> gpurun_out/bench6.err
python tools/prof_step.py > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ax_v5" -s 2 -c 1 -o gpurun_out/prof_r1e python tools/prof_step.py > gpurun_out/ncu2.log 2>&1
