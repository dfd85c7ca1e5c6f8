#!/bin/bash
# Assembly iteration on the GPU box: parity, A/B timing against libmm_base.so on c2/c3, ncu captures.
timeout 900 python -m pytest tests/test_gpu_zeroing.py tests/test_gpu_parity.py -q -x > gpurun_out/ab_pytest.log 2>&1
tail -3 gpurun_out/ab_pytest.log
for c in c2 c3; do
  for i in 1 2; do
    echo "new:  $(timeout 300 python tools/time_asm.py $c 30 2>&1 | tail -1)"
    echo "base: $(timeout 300 python tools/time_asm.py $c 30 paper_2604_19286_b200/libmm_base.so 2>&1 | tail -1)"
  done
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_asm_o1t -s 2 -c 1 -f -o gpurun_out/ab_o1t python tools/time_asm.py c2 1 > gpurun_out/ab_ncu.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_asm_o2t -s 2 -c 1 -f -o gpurun_out/ab_o2t python tools/time_asm.py c3 1 >> gpurun_out/ab_ncu.log 2>&1
tail -2 gpurun_out/ab_ncu.log
