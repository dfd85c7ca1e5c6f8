nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for L in libmm libmm_fr4 libmm_fr5 libmm libmm_fr4; do echo "== $L"; MM_SORT_TIMERS=1 timeout 300 python tools/time_sort_big.py 3 paper_2604_19286_b200/$L.so 2>&1 | grep -v "^\[mm sort\]" ; done
