mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "gs or window or rod" > gpurun_out/j13_tests.log 2>&1; echo "parity $?" > gpurun_out/j13_summary.txt
tail -1 gpurun_out/j13_tests.log >> gpurun_out/j13_summary.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"gs_chunk|gs_classes" -s 1 -c 1 -o gpurun_out/j13_chunk_big python tools/prof_step.py --solves 0 --ax 3 --ez 128 > gpurun_out/j13_1.log 2>&1; echo "chunk big $?" >> gpurun_out/j13_summary.txt
S=gpurun_out/j13_summary.txt
for pf in 1 0 1 0; do
  NEK_GS_CHUNK=$pf timeout 300 python bench.py --no-cpu-baseline --no-peaks > gpurun_out/j13_b.json 2>gpurun_out/j13_b.err; echo "bench pf=$pf $?" >> $S
  python -c "import json;d=json.loads(open('gpurun_out/j13_b.json').read().strip().splitlines()[-1]);print('pf=$pf', d['value'], d['ms_per_step'], d['kernel_ms_per_step']['gs_ms'], 'axgs', d['ax_gs']['gs_kernel']['avg_launch_ms'], d['ax_gs']['gs_kernel']['frac'], 'big', d['beyond_l2']['gs']['avg_launch_ms'], d['beyond_l2']['gs']['frac'], d['beyond_l2']['ax_gs']['frac'])" >> $S
done
