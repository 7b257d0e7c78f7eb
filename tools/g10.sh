mkdir -p gpurun_out
NEK_LIB_VARIANT=checked timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/g10_checked.log 2>&1
echo "checked exit $?" >> gpurun_out/g10_summary.txt
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/g10_gpu.log 2>&1
echo "gpu exit $?" >> gpurun_out/g10_summary.txt
