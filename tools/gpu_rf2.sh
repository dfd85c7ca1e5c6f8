nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_recfirst.py -x -q > gpurun_out/pytest_rf.log 2>&1; echo pytest_rf $?
tail -5 gpurun_out/pytest_rf.log
MM_SORT_TIMERS=1 timeout 600 python tools/time_sort_big.py 3 > gpurun_out/bigph.log 2>&1; echo big $?
grep -v "^\[mm sort\]" gpurun_out/bigph.log; grep "^\[mm sort\]" gpurun_out/bigph.log | sed -n '2p;8p;14p'
