mkdir -p gpurun_out
S=gpurun_out/j6_summary.txt; : > $S
n=${1:-2}
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29631 tools/mgpu_check.py > gpurun_out/j6_mgpu$n.log 2>&1; echo "mgpu $?" >> $S
tail -3 gpurun_out/j6_mgpu$n.log >> $S
for d in 1 0 1 0; do
  NEK_DEFER=$d timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 29632 bench.py --gpus $n --no-pmg --no-cpu-baseline --no-peaks > gpurun_out/j6_b$n_$d.json 2> gpurun_out/j6_b$d.err; echo "bench defer=$d $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j6_b$n_$d.json').read().strip().splitlines()[-1]);print('defer=$d', d['value'], d['ms_per_step'], d['kernel_ms_per_step'])" >> $S
done
