#!/bin/bash
# NEXT-4 iteration: GPU parity of moments / gather, timing vs libmm_base.so on the c2 handle.
timeout 900 python -m pytest tests/test_gpu_next4.py -q -x > gpurun_out/n4_pytest.log 2>&1; echo "next4 tests rc $?"
tail -2 gpurun_out/n4_pytest.log
for lib in - paper_2604_19286_b200/libmm_base.so; do
  echo "lib $lib: $(timeout 300 python tools/time_next4.py $lib 2>&1 | tail -3 | tr '\n' ' ')"
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"k_moments|k_gather" -s 3 -c 3 -f -o gpurun_out/n4 python tools/time_next4.py - > gpurun_out/n4_ncu.log 2>&1
tail -1 gpurun_out/n4_ncu.log
