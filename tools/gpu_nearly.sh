nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
MM_SORT_TIMERS=1 timeout 300 python tools/time_sort_nearly.py > gpurun_out/nearly.log 2>&1; echo nearly $?
grep -v "^\[mm sort\]" gpurun_out/nearly.log; grep "^\[mm sort\]" gpurun_out/nearly.log | sed -n '5p;20p'
MM_SORT_TIMERS=1 MM_SORT_RECFIRST_MIN=1 timeout 300 python tools/time_sort_nearly.py > gpurun_out/nearly_rf.log 2>&1; echo nearly_rf $?
grep -v "^\[mm sort\]" gpurun_out/nearly_rf.log; grep "^\[mm sort\]" gpurun_out/nearly_rf.log | sed -n '5p;20p'
timeout 600 ncu --set full --clock-control none -k regex:"k_key|k_place|k_fix_warp|k_scatter" -s 20 -c 4 -f -o gpurun_out/prof_nearly python tools/time_sort_nearly.py > /dev/null 2>&1; echo ncu $?
