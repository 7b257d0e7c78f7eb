T="python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29531"
timeout 600 $T tools/mgpu_check.py > gpurun_out/fold_check.log 2>&1; grep '^{' gpurun_out/fold_check.log | tail -1 | cut -c1-200; echo
NEK_CONCURRENT_BND=0 timeout 600 $T tools/mgpu_check.py > gpurun_out/fold_check_so.log 2>&1; grep '^{' gpurun_out/fold_check_so.log | tail -1 | cut -c1-200; echo
NEK_FOLD=0 timeout 600 $T tools/mgpu_check.py > gpurun_out/fold_check_f0.log 2>&1; grep '^{' gpurun_out/fold_check_f0.log | tail -1 | cut -c1-200; echo
timeout 900 python -m pytest tests/test_multigpu.py -x -q 2>&1 | tail -2
