timeout 900 python -m pytest tests/test_gpu_pmg.py -x -q > gpurun_out/pytest_pmg.log 2>&1; tail -20 gpurun_out/pytest_pmg.log
timeout 300 python tools/pmg_bench.py --ez 16 > gpurun_out/pmgb64.jsonl 2>&1; tail -1 gpurun_out/pmgb64.jsonl
timeout 300 python tools/pmg_bench.py --ez 16 --precision 1 > gpurun_out/pmgb32.jsonl 2>&1; tail -1 gpurun_out/pmgb32.jsonl
timeout 300 python tools/pmg_profile.py --precision 1 > gpurun_out/pmg_prof32.json 2> gpurun_out/pmg_prof.err; cat gpurun_out/pmg_prof32.json | python -c "
import sys,json; d=json.loads(sys.stdin.read()); print(d['us_per_vcycle_kernels'], d['launches_per_vcycle'])
for r in d['by_kernel'][:16]: print(r)"
echo done
