#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_resort.py tests/test_gpu_async_sort.py -q -x > gpurun_out/resort_pytest.log 2>&1; echo "resort tests rc $?"; tail -15 gpurun_out/resort_pytest.log
timeout 300 python tools/time_resort.py > gpurun_out/resort_time.log 2>&1; cat gpurun_out/resort_time.log | tail -6
