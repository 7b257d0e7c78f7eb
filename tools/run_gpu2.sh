mkdir -p gpurun_out
S=gpurun_out/j26_summary.txt; : > $S
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "prefetch or variants or window or config2 or rod or config3" > gpurun_out/j26_tests.log 2>&1; echo "tests $?" >> $S
tail -1 gpurun_out/j26_tests.log >> $S
NEK_LIB_VARIANT=checked timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "prefetch or variants" > gpurun_out/j26_tests_c.log 2>&1; echo "checked $?" >> $S
tail -1 gpurun_out/j26_tests_c.log >> $S
