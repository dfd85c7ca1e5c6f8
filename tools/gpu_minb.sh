nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for M in 5 4 5 4 6; do echo "minb $M"; MM_O1T_MINB=$M timeout 300 python tools/time_variant2.py paper_2604_19286_b200/libmm.so c2 2>&1 | tail -1; done
