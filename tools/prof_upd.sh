timeout 300 python tools/prof_step.py --solves 1 --iters 4 --ax 0 > gpurun_out/prof_plain.log 2>&1; tail -2 gpurun_out/prof_plain.log
timeout 900 ncu --set full --import-source on -k regex:"pcg_update_fused|gs_classes" -c 4 -o gpurun_out/upd_full -f python tools/prof_step.py --solves 1 --iters 4 --ax 0 > gpurun_out/prof_ncu.log 2>&1; tail -3 gpurun_out/prof_ncu.log
