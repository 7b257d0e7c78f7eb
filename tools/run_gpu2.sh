mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"makef_mma" -s 2 -c 1 -o gpurun_out/r2_makef_mma python tools/makef_bench.py > gpurun_out/j1_ncu.log 2>&1; echo "ncu $?" >> gpurun_out/j1_summary.txt
