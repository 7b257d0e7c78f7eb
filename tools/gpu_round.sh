R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
S=$(date +%s); python bench.py > gpurun_out/bdef1.json 2> gpurun_out/bdef1.err; tail -1 gpurun_out/bdef1.err; echo "bench1 $(( $(date +%s) - S )) s"
$R --master-port 29571 bench.py --gpus 4 > gpurun_out/bdef4.json 2> gpurun_out/bdef4.err; tail -1 gpurun_out/bdef4.err
python bench.py --impl reference > gpurun_out/bref1.json 2> gpurun_out/bref1.err; tail -1 gpurun_out/bref1.err
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
for f in bdef1 bdef4 bref1; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f', {k: d.get(k) for k in ('value','e2e','pcg_iter_per_s','gpu_launches','impl')}, d.get('roofline',{}) and d['roofline']['frac'], d.get('cpu_baseline'))"; done
echo done
