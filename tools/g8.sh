mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gs_classes_kernel|pcg_update_fused|ax_v5" -s 9 -c 4 -o gpurun_out/r2_big python tools/prof_step.py --ez 128 --solves 1 --iters 3 --ax 2 > gpurun_out/g8_ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/g8_summary.txt
