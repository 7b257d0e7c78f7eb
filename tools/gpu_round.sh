set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench8.json 2> gpurun_out/bench8.err
python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline > gpurun_out/bench8g.json 2>> gpurun_out/bench8.err
python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/prof_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum --cache-control none --clock-control none --csv --log-file gpurun_out/launches_warm.csv python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/ncu1.log 2>&1
ncu --set full --cache-control none --clock-control none --import-source on -k regex:"gs_classes|update_fused" -s 6 -c 2 -o gpurun_out/prof_r1f python tools/prof_step.py --solves 2 --iters 10 > gpurun_out/ncu2.log 2>&1
