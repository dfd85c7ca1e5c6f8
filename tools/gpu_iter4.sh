#!/bin/bash
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_zeroing.py -q -x > gpurun_out/it4_pytest.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/it4_pytest.log
for i in 1 2; do echo "c2: $(timeout 300 python tools/time_asm.py c2 40 2>&1 | tail -1)"; done
echo "c4: $(timeout 300 python tools/time_c4.py 1 5 2>&1 | tail -1) / $(timeout 300 python tools/time_c4.py 2 5 2>&1 | tail -1)"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_asm_o1t -s 2 -c 1 -f -o gpurun_out/it4_o1t python tools/time_asm.py c2 1 > /dev/null 2>&1; echo "ncu rc $?"
