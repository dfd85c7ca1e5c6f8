#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_sort_tf32.py tests/test_gpu_resort.py tests/test_gpu_async_sort.py -q -x -k "sort or resort or mixed or scalar_handle" > gpurun_out/scat_pytest.log 2>&1; echo "sort tests rc $?"; tail -1 gpurun_out/scat_pytest.log
MM_SORT_TIMERS=1 timeout 300 python tools/time_sort.py c2 5 2>&1 | grep "mm sort" | tail -2
timeout 300 python tools/time_sort.py c2 20 2>&1 | tail -1
MM_SORT_TIMERS=1 timeout 600 python tools/time_sort_big.py 2 - 2>&1 | grep -v "^\[mm sort\]" | tail -3
