mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_makef.py -q > gpurun_out/i1_makef.log 2>&1; echo "makef $?" >> gpurun_out/i1_summary.txt
timeout 300 python tools/makef_bench.py > gpurun_out/i1_makef_bench.log 2>&1; echo "mkbench $?" >> gpurun_out/i1_summary.txt
NEK_MAKEF_VARIANT=3 timeout 300 python tools/makef_bench.py > gpurun_out/i1_makef_bench3.log 2>&1; echo "mkbench3 $?" >> gpurun_out/i1_summary.txt
timeout 600 python bench.py --mesh rod --no-pmg --no-beyond --no-cpu-baseline --steps 5 > gpurun_out/h1_rod.json 2> gpurun_out/h1_rod.err; echo "rod $?" >> gpurun_out/i1_summary.txt
timeout 600 python bench.py --mesh rod --h2 100 --no-pmg --no-beyond --no-cpu-baseline --steps 5 > gpurun_out/h1_rod_h.json 2> gpurun_out/h1_rod_h.err; echo "rodh $?" >> gpurun_out/i1_summary.txt
timeout 900 python bench.py --mesh cfg3 --no-pmg --no-beyond --no-cpu-baseline --steps 3 > gpurun_out/h1_cfg3.json 2> gpurun_out/h1_cfg3.err; echo "cfg3 $?" >> gpurun_out/i1_summary.txt
timeout 900 python tools/nsweep.py > gpurun_out/h1_nsweep.log 2>&1; echo "nsweep $?" >> gpurun_out/i1_summary.txt
