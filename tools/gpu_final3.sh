# final verification of the committed state on one GPU: the driver's round-end commands
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/fin_pytest.log 2>&1; tail -3 gpurun_out/fin_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; tail -c 300 gpurun_out/fin_bench.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; tail -c 200 gpurun_out/fin_ref.json
