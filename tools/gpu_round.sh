R="python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1"
timeout 600 $R --master-port 29530 tools/mgpu_check.py > gpurun_out/mgpu4.log 2>&1; tail -1 gpurun_out/mgpu4.log | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['ok'], {k:(v['ok'], v['pmg']) for k,v in d['cases'].items()})"
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/b1.json 2>gpurun_out/b1.err
python -c "import json;d=json.loads(open('gpurun_out/b1.json').read().strip().splitlines()[-1]);print(d['value'], d['pmg'], d['cpu_baseline'])"
for ez in 16 128; do
timeout 300 $R --master-port 2953$((ez % 7)) bench.py --gpus 4 --steps 10 --warmup 3 --ez $ez > gpurun_out/b4_ez$ez.json 2> gpurun_out/b4.err
done
timeout 600 $R --master-port 29551 bench.py --gpus 4 --steps 3 --warmup 3 --mesh rod > gpurun_out/b4_rod.json 2>> gpurun_out/b4.err
for f in b4_ez16 b4_ez128 b4_rod; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f',round(d['value'],2),round(d['pcg_iter_per_s']),d['clocks']['sm_mhz'], d['pmg'])"; done
echo done
