mkdir -p gpurun_out
timeout 600 ncu --set full --cache-control none --clock-control none --import-source on -k regex:"gs_classes_kernel|pcg_update_fused|ax_v5" -s 30 -c 6 -o gpurun_out/r2_step_warm python tools/prof_step.py --solves 2 --iters 8 --ax 0 > gpurun_out/g4_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/g4_summary.txt
