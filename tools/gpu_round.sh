R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 900 python -m pytest tests -q -m gpu -x > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 $R --master-port 29530 tools/mgpu_check.py > gpurun_out/mgpu4.log 2>&1; tail -1 gpurun_out/mgpu4.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['ok'], {k:(v['ok'], v['pmg']) for k,v in d['cases'].items()})"
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b1.json 2>gpurun_out/b1.err
python -c "import json;d=json.loads(open('gpurun_out/b1.json').read().strip().splitlines()[-1]);print(d['value'], d['pmg'])"
timeout 300 python tools/pmg_profile.py --precision 1 > gpurun_out/pmg_prof32.json 2> gpurun_out/pmg_prof.err; cat gpurun_out/pmg_prof32.json | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['us_per_vcycle_kernels'], d['launches_per_vcycle'])
for r in d['by_kernel'][:8]: print(r)"
echo done
