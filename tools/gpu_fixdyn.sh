nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_resort.py tests/test_gpu_recfirst.py tests/test_gpu_async_sort.py -x -q -k "sort or resort or recfirst" > gpurun_out/pytest_fix.log 2>&1; echo pytest_fix $?
tail -2 gpurun_out/pytest_fix.log
MM_SORT_TIMERS=1 timeout 300 python tools/time_sort_nearly.py > gpurun_out/nearly_dyn.log 2>&1; grep -v "^\[mm sort\]" gpurun_out/nearly_dyn.log; grep "^\[mm sort\]" gpurun_out/nearly_dyn.log | sed -n '5p;20p'
for L in libmm libmm_fix0 libmm libmm_fix0; do echo "== $L"; MM_SORT_TIMERS=1 timeout 300 python tools/time_sort_big.py 3 paper_2604_19286_b200/$L.so > gpurun_out/big_$L.log 2>&1; grep -v "^\[mm sort\]" gpurun_out/big_$L.log; grep "^\[mm sort\]" gpurun_out/big_$L.log | sed -n '3p;9p'; done
