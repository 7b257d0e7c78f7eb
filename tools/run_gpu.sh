# GPU validation sequence used at the end of round 2 (gpurun -- bash tools/run_gpu.sh <mode>):
#   bench   the default bench line + the reference arm
#   tests   pytest -m gpu (production library), then with the checked build
#   ncu     launch list of the default bench and one --set full capture of the step's kernels
mkdir -p gpurun_out
mode=${1:-bench}
tag=${2:-v}
if [ "$mode" = bench ]; then
  timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench $?" >> gpurun_out/${tag}_summary.txt
  timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref $?" >> gpurun_out/${tag}_summary.txt
fi
if [ "$mode" = tests ]; then
  timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_gpu.log 2>&1; echo "gpu $?" >> gpurun_out/${tag}_summary.txt
  NEK_LIB_VARIANT=checked timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${tag}_checked.log 2>&1; echo "checked $?" >> gpurun_out/${tag}_summary.txt
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${tag}_smoke.log 2>&1; echo "smoke $?" >> gpurun_out/${tag}_summary.txt
fi
if [ "$mode" = ncu ]; then
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv --log-file gpurun_out/${tag}_launches.csv python bench.py --steps 2 --warmup 1 --no-pmg --no-peaks --no-cpu-baseline --no-beyond > gpurun_out/${tag}_ncu_launch.log 2>&1; echo "launches $?" >> gpurun_out/${tag}_summary.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"gs_chunk|pcg_update|ax_v5" -s 30 -c 3 -o gpurun_out/${tag}_full python tools/prof_step.py --solves 2 --iters 8 --ax 0 > gpurun_out/${tag}_ncu_full.log 2>&1; echo "full $?" >> gpurun_out/${tag}_summary.txt
fi
if [ "$mode" = mgpu ]; then
  n=${3:-2}
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/${tag}_mgpu${n}.log 2>&1; echo "mgpu $?" >> gpurun_out/${tag}_summary.txt
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus $n --no-pmg > gpurun_out/${tag}_bench${n}.json 2> gpurun_out/${tag}_bench${n}.err; echo "bench$n $?" >> gpurun_out/${tag}_summary.txt
fi
