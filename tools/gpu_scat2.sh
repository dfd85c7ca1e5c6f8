#!/bin/bash
for i in 1 2 3; do
echo "new:  $(timeout 300 python tools/time_sort.py c2 30 2>&1 | tail -1)"
echo "prev: $(timeout 300 python tools/time_sort.py c2 30 paper_2604_19286_b200/libmm_prev.so 2>&1 | tail -1)"
done
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
