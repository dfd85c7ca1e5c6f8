set -x
python -m pytest tests/test_gpu_parity.py -x -q -k "sort or parity_uniform or errors or empty or special or large or c4 or mixed or scalar_handle" 2>&1 | tail -4
for i in 1 2; do
python tools/time_sort.py c2 30 tools/libmm_prev.so
python tools/time_sort.py c2 30
done
python tools/time_sort.py c3 20 tools/libmm_prev.so
python tools/time_sort.py c3 20
MM_SORT_TIMERS=1 python tools/time_sort.py c2 3 2>&1 | tail -2
MM_SORT_TIMERS=1 python tools/time_sort.py c2 3 tools/libmm_prev.so 2>&1 | tail -2
python tools/time_sort_nearly.py
