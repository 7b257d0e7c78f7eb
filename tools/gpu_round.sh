for v in 0 1; do NEK_MAKEF_VARIANT=$v timeout 300 python tools/makef_bench.py > gpurun_out/makef_v$v.json 2>&1; echo "v$v"; cat gpurun_out/makef_v$v.json; done
