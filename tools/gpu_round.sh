set -x
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1
python bench.py --steps 10 --warmup 3 > gpurun_out/bench10.json 2> gpurun_out/bench10.err
for v in 0 9; do python bench.py --steps 10 --warmup 3 --graph --no-cpu-baseline --variant $v > gpurun_out/bench10g_v$v.json 2>> gpurun_out/bench10.err; done
python bench.py --steps 5 --warmup 3 --graph --no-cpu-baseline --ez 128 > gpurun_out/bench10g_ez128.json 2>> gpurun_out/bench10.err
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --ez 128 > gpurun_out/bench10_ez128.json 2>> gpurun_out/bench10.err
python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/bench_small.json 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bench_r1.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu1.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"ax_v5|gs_classes|update_fused" -s 40 -c 3 -o gpurun_out/prof_bench_r1 python bench.py --steps 2 --warmup 3 --no-cpu-baseline > gpurun_out/ncu2.log 2>&1
