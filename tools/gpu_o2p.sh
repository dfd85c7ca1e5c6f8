#!/bin/bash
# o2t pair variant (MM_O2T_PAIR=1): order-2 parity, A/B timing vs the per-bin kernel, ncu.
MM_O2T_PAIR=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_parity_sort_tf32.py tests/test_gpu_zeroing.py -q -x -k "order2 or o2 or 2- or -2 or full_size or slab or lattice or c3 or accumulate or tsc or zero" > gpurun_out/o2p_pytest.log 2>&1; echo "parity rc $?"
grep -E "passed|failed|Error" gpurun_out/o2p_pytest.log | head -5
for i in 1 2; do
echo "c3 base: $(timeout 120 python tools/time_asm.py c3 20 2>&1 | tail -1)"
echo "c3 pair: $(MM_O2T_PAIR=1 timeout 120 python tools/time_asm.py c3 20 2>&1 | tail -1)"
done
MM_O2T_PAIR=1 timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_asm_o2p -s 2 -c 1 -f -o gpurun_out/o2p python tools/time_asm.py c3 1 > /dev/null 2>&1; echo "ncu rc $?"
