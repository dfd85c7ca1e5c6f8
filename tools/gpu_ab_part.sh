MM_SORT_PART_NP=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "sort or parity_uniform or errors or empty or special or mixed or scalar_handle or slab or clustered or cell_ordered or lattice" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "c4" 2>&1 | tail -2
python tools/c4_sort_phases.py tools/libmm_prev.so
python tools/c4_sort_phases.py
MM_SORT_TIMERS=1 python tools/c4_sort_phases.py 2>&1 | tail -3
python tools/time_sort.py c2 20
MM_SORT_PART_NP=0 python tools/time_sort.py c2 20
MM_SORT_PART_NP=0 MM_SORT_TIMERS=1 python tools/time_sort.py c2 3 2>&1 | tail -2
