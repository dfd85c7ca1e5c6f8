#!/bin/bash
# sort phases beyond L2 (bucketed vs direct), NEXT-4 timing, gather parity.
timeout 300 python -m pytest tests/test_gpu_next4.py -q -x > gpurun_out/it3_pytest.log 2>&1; echo "next4 tests rc $?"; tail -1 gpurun_out/it3_pytest.log
echo "next4: $(timeout 300 python tools/time_next4.py - 2>&1 | tail -3 | tr '\n' ' ')"
MM_SORT_TIMERS=1 MM_SORT_BKT_MIN=1 timeout 600 python tools/time_sort_big.py 2 - > gpurun_out/it3_bkt.log 2>&1
MM_SORT_TIMERS=1 timeout 600 python tools/time_sort_big.py 2 - > gpurun_out/it3_direct.log 2>&1
grep "mm sort" gpurun_out/it3_bkt.log | tail -3
grep "mm sort" gpurun_out/it3_direct.log | tail -3
MM_SORT_BKT_MIN=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio --clock-control none -k regex:"k_bkt|k_fix_warp|k_key|k_scatter" -c 12 --csv --log-file gpurun_out/it3_bkt_ncu.csv python tools/time_sort_big.py 1 - > /dev/null 2>&1; echo "ncu rc $?"
