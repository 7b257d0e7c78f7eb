timeout 900 python -m pytest tests/test_gpu_makef.py -x -q > gpurun_out/pytest_makef.log 2>&1; tail -3 gpurun_out/pytest_makef.log
timeout 300 python tools/makef_bench.py > gpurun_out/makef_b.json 2>&1; cat gpurun_out/makef_b.json
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/b1.json 2>gpurun_out/b1.err; tail -1 gpurun_out/b1.json | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['makef'], d['projection'], d['pmg']['fp32'])"
tail -3 gpurun_out/b1.err
echo done
