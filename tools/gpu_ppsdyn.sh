nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for L in libmm libmm_pps4 libmm_pps8 libmm_pps16 libmm libmm_pps8; do
  for O in 1 2; do echo "$L o$O $(timeout 300 python tools/time_c4.py $O 6 paper_2604_19286_b200/$L.so 2>&1 | tail -1)"; done
done
