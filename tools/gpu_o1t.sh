#!/bin/bash
# o1t A/B: base library vs the new kernel with the memset (MM_ZERO_O1=0) and with in-kernel zeroing (=1).
timeout 900 python -m pytest tests/test_gpu_zeroing.py -q -x > gpurun_out/o1t_pytest.log 2>&1
MM_ZERO_O1=1 timeout 900 python -m pytest tests/test_gpu_zeroing.py tests/test_gpu_parity.py -q -x -k "zero or uniform or lattice or slab or c1 or full_size" >> gpurun_out/o1t_pytest.log 2>&1
grep -E "passed|failed" gpurun_out/o1t_pytest.log
for i in 1 2; do
  echo "new memset: $(MM_ZERO_O1=0 timeout 300 python tools/time_asm.py c2 40 2>&1 | tail -1)"
  echo "new zero:   $(MM_ZERO_O1=1 timeout 300 python tools/time_asm.py c2 40 2>&1 | tail -1)"
  echo "base:       $(timeout 300 python tools/time_asm.py c2 40 paper_2604_19286_b200/libmm_base.so 2>&1 | tail -1)"
done
MM_ZERO_O1=0 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_asm_o1t -s 2 -c 1 -f -o gpurun_out/o1t_memset python tools/time_asm.py c2 1 > gpurun_out/o1t_ncu.log 2>&1
tail -1 gpurun_out/o1t_ncu.log
