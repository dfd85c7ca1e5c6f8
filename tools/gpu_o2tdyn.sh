nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for L in libmm libmm_o2t2 libmm_o2t4 libmm libmm_o2t2 libmm_o2t4; do timeout 300 python tools/time_variant2.py paper_2604_19286_b200/$L.so c3 2>&1 | tail -1; done
