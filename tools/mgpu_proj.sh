# 2 GPUs: default bench (pMG, projection, makef sections) with and without the folded bookkeeping
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29551"
for f in 1 0; do
  NEK_FOLD=$f timeout 600 $T bench.py --gpus 2 --steps 3 --no-peaks > gpurun_out/pj_f$f.json 2> gpurun_out/pj_f$f.err
  echo "fold=$f rc=$?"; grep -h "NekError" gpurun_out/pj_f$f.err | head -2; tail -c 300 gpurun_out/pj_f$f.json; echo
done
