#!/bin/bash
MM_SORT_TIMERS=1 timeout 300 python tools/time_resort.py > gpurun_out/resort_t2.log 2>&1
grep "mm sort" gpurun_out/resort_t2.log | awk '{c[$0]++} END{for(k in c) print c[k], k}' | sort -rn | head -12
