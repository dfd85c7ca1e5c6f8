#!/bin/bash
# o2t iteration: parity (order-2 parity), A/B timing of the ticket-order z block vs libmm_base.so, ncu.
timeout 900 python -m pytest tests/test_gpu_zeroing.py tests/test_gpu_parity.py tests/test_gpu_parity_sort_tf32.py tests/test_gpu_next4.py -q -x -k "zero or order2 or o2 or 2- or -2 or full_size or slab or lattice or c3 or accumulate or tsc" > gpurun_out/o2t_pytest.log 2>&1; echo "parity rc $?"
grep -E "passed|failed|Error" gpurun_out/o2t_pytest.log | head
for i in 1 2; do
echo "c3 base:   $(timeout 120 python tools/time_asm.py c3 20 paper_2604_19286_b200/libmm_base.so 2>&1 | tail -1)"
for zb in 0 4 8 16; do
echo "c3 zb $zb: $(MM_O2T_ZB=$zb timeout 120 python tools/time_asm.py c3 20 2>&1 | tail -1)"
done
done
timeout 300 ncu --set full --clock-control none --import-source on -k regex:k_asm_o2t -s 2 -c 1 -f -o gpurun_out/o2t_zb python tools/time_asm.py c3 1 > gpurun_out/o2t_ncu.log 2>&1
tail -1 gpurun_out/o2t_ncu.log
