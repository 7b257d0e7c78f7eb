mkdir -p gpurun_out
bash tools/run_gpu.sh tests k8
bash tools/run_gpu.sh bench k8
bash tools/run_gpu.sh ncu k8
