nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
MM_SORT_TIMERS=1 timeout 600 python tools/c4_sort_phases.py > gpurun_out/c4ph.log 2>&1; echo c4ph $?
cat gpurun_out/c4ph.log | tail -20
MM_SORT_TIMERS=1 timeout 600 python tools/time_sort_big.py 2 > gpurun_out/bigph.log 2>&1; echo big $?
tail -20 gpurun_out/bigph.log
MM_SORT_TIMERS=1 timeout 600 python tools/time_sort.py c2 3 > gpurun_out/c2ph.log 2>&1; echo c2 $?
tail -12 gpurun_out/c2ph.log
