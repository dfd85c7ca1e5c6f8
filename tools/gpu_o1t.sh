#!/bin/bash
# o1t iteration on the GPU box: parity, A/B timing against the round-1 library, one ncu capture.
timeout 600 python -m pytest tests/test_gpu_parity_sort_tf32.py -q -x -k "store_first" > gpurun_out/o1t_pytest.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "c1 or uniform or lattice or full_size" >> gpurun_out/o1t_pytest.log 2>&1
grep -E "passed|failed" gpurun_out/o1t_pytest.log
for i in 1 2; do
  echo "new: $(timeout 300 python tools/time_asm.py c2 30 2>&1 | tail -1)"
  echo "r1:  $(timeout 300 python tools/time_asm.py c2 30 paper_2604_19286_b200/libmm_r1.so 2>&1 | tail -1)"
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_asm_o1t -s 2 -c 1 -f -o gpurun_out/o1t_v6 python tools/time_asm.py c2 1 >> gpurun_out/o1t_ncu.log 2>&1
tail -1 gpurun_out/o1t_ncu.log
