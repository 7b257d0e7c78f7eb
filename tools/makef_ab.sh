# makef with the L2 prefetch of the next element's lattice factors (per-component kernel and merged variant)
for v in 0 1; do NEK_MAKEF_VARIANT=$v timeout 300 python tools/makef_bench.py --reps 10 2>&1 | tail -1 | cut -c1-400; done
timeout 600 python -m pytest tests/test_gpu_makef.py -x -q 2>&1 | tail -2
