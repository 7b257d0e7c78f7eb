# Round artefacts on 1 GPU: default bench line, launch list of the same command, ncu --set full of the
# PCG kernels at config 2, config 3 strong-scaling point and the rod bundle (config 4) on one GPU
timeout 600 python bench.py > gpurun_out/f_bench.json 2> gpurun_out/f_bench.err; tail -c 600 gpurun_out/f_bench.json; echo
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/f_launches.csv python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-pmg --no-peaks > gpurun_out/f_ncu_launch.log 2>&1; tail -2 gpurun_out/f_ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ax_v5_kernel|gs_classes_kernel|pcg_update_fused_kernel" -s 6 -c 3 -o gpurun_out/f_full -f python tools/prof_step.py --solves 2 --iters 5 --ax 3 > gpurun_out/f_ncu_full.log 2>&1; tail -2 gpurun_out/f_ncu_full.log
timeout 600 python bench.py --mesh cfg3 --no-pmg --no-peaks --no-cpu-baseline --steps 3 > gpurun_out/f_cfg3.json 2> gpurun_out/f_cfg3.err; tail -c 300 gpurun_out/f_cfg3.json; echo
timeout 600 python bench.py --mesh rod --no-pmg --no-peaks --no-cpu-baseline --steps 3 > gpurun_out/f_rod.json 2> gpurun_out/f_rod.err; tail -c 300 gpurun_out/f_rod.json; echo
