python -m pytest tests/test_gpu_parity.py -x -q -k "c4 or parity_uniform or clustered or lattice or scalar_handle or c1 or slab or species or accumulate or nonunit or special" 2>&1 | tail -3
for i in 1 2; do
MM_ASM_PPS1=1 python tools/time_c4.py 1 5
python tools/time_c4.py 1 5
done
