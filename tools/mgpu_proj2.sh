# 2 GPUs: which part of the folded path breaks the projection sequence (L2 carve-out off / eager launches)
T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29571"
run() { tag=$1; shift
  env "$@" timeout 300 $T bench.py --gpus 2 --steps 2 --warmup 3 --no-peaks > gpurun_out/pj2_$tag.json 2> gpurun_out/pj2_$tag.err
  echo "$tag rc=$?"; grep -h "NekError" gpurun_out/pj2_$tag.err | head -1; tail -c 250 gpurun_out/pj2_$tag.json | head -c 200; echo; }
run f1k0 NEK_FOLD=1 NEK_L2KEEP=0
run f1ng NEK_FOLD=1 NEK_NO_GRAPH=1
