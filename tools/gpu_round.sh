for i in 1 2 3; do timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/b1_$i.json 2>/dev/null; done
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variant 10 > gpurun_out/b1_v10.json 2>/dev/null
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --variant 8 > gpurun_out/b1_v8.json 2>/dev/null
for f in b1_1 b1_2 b1_3 b1_v10 b1_v8; do python -c "
import json;d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]);print('$f',round(d['value'],2),round(d['pcg_iter_per_s']),d['clocks'], d['kernel_ms_per_step'])"; done
echo done
