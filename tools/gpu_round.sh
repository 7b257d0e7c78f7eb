timeout 600 python tools/nsweep.py 3 4 5 6 8 9 > gpurun_out/nsweep_v6.jsonl 2> gpurun_out/nsweep_v6.err
NSWEEP_VARIANT=1 timeout 600 python tools/nsweep.py 3 5 9 > gpurun_out/nsweep_v0.jsonl 2>> gpurun_out/nsweep_v6.err
cat gpurun_out/nsweep_v6.jsonl gpurun_out/nsweep_v0.jsonl
echo done
