#!/bin/bash
# Round-2 iteration: new GPU tests (async sort, bucketed sort, NEXT-4, zeroing), NEXT-4 and
# big-sort timing against libmm_base.so, a short bench.
timeout 600 python -m pytest tests/test_gpu_async_sort.py tests/test_gpu_next4.py tests/test_gpu_zeroing.py -q -x > gpurun_out/it2_pytest.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/it2_pytest.log
timeout 1500 python -m pytest tests/test_gpu_sort_bucketed.py -q -x > gpurun_out/it2_bkt.log 2>&1; echo "bucketed rc $?"; tail -2 gpurun_out/it2_bkt.log
timeout 900 python -m pytest tests/test_gpu_parity_sort_tf32.py -q -x -k "full_size" > gpurun_out/it2_full.log 2>&1; echo "full-size rc $?"; tail -2 gpurun_out/it2_full.log
echo "next4 new:  $(timeout 300 python tools/time_next4.py - 2>&1 | tail -3 | tr '\n' ' ')"
echo "next4 base: $(timeout 300 python tools/time_next4.py paper_2604_19286_b200/libmm_base.so 2>&1 | tail -3 | tr '\n' ' ')"
echo "big sort new (bucketed): $(timeout 600 python tools/time_sort_big.py 5 - 2>&1 | tail -3 | tr '\n' ' ')"
echo "big sort new (direct):   $(MM_SORT_BKT_MIN=2000000000 timeout 600 python tools/time_sort_big.py 5 - 2>&1 | tail -3 | tr '\n' ' ')"
SECONDS=0; timeout 900 python bench.py --steps 100 --no-cpu-baseline > gpurun_out/it2_bench.json 2> gpurun_out/it2_bench.err; echo "bench rc $? wall $SECONDS"
