#!/bin/bash
# o2t iteration: parity (zeroing + order-2 parity), A/B timing of the z-segment variants vs libmm_base.so, ncu.
timeout 300 python -m pytest tests/test_gpu_zeroing.py -q -x > gpurun_out/o2t_pytest.log 2>&1; echo "zeroing rc $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_sort_tf32.py tests/test_gpu_next4.py -q -x -k "order2 or o2 or 2- or -2 or full_size or slab or lattice or c3 or accumulate or tsc" >> gpurun_out/o2t_pytest.log 2>&1; echo "parity rc $?"
grep -E "passed|failed|Error" gpurun_out/o2t_pytest.log | head
echo "c3 base: $(timeout 120 python tools/time_asm.py c3 20 paper_2604_19286_b200/libmm_base.so 2>&1 | tail -1)"
for seg in 4 8 16; do
  echo "c3 seg $seg zero:   $(MM_O2T_SEG=$seg timeout 120 python tools/time_asm.py c3 20 2>&1 | tail -1)"
  echo "c3 seg $seg memset: $(MM_O2T_SEG=$seg MM_ZERO_O2=0 timeout 120 python tools/time_asm.py c3 20 2>&1 | tail -1)"
done
echo "c2 new:  $(timeout 120 python tools/time_asm.py c2 40 2>&1 | tail -1)"
echo "c2 base: $(timeout 120 python tools/time_asm.py c2 40 paper_2604_19286_b200/libmm_base.so 2>&1 | tail -1)"
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_asm_o2t -s 2 -c 1 -f -o gpurun_out/o2t_ws python tools/time_asm.py c3 1 > gpurun_out/o2t_ncu.log 2>&1
tail -1 gpurun_out/o2t_ncu.log
