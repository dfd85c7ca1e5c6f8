nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for L in libmm_dyn2 libmm_dyn4 libmm_dyn8 libmm_dyn16 libmm_dyn2 libmm_dyn4 libmm_dyn8 libmm_dyn16; do timeout 300 python tools/time_variant2.py paper_2604_19286_b200/$L.so c2 2>&1 | tail -1; done
