for lib in paper_2604_19286_b200/libmm.so paper_2604_19286_b200/libmm_cs.so; do
  echo $lib
  timeout 300 python tools/time_sort.py c2 30 $lib
  MM_SORT_TIMERS=1 timeout 300 python tools/time_sort.py c2 3 $lib 2>&1 | tail -2
done
