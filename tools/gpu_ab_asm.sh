python -m pytest tests/test_gpu_parity.py -x -q -k "parity_uniform or lattice or c1 or full_size or species or nonunit or accumulate or slab or cell_ordered or special" 2>&1 | tail -2
for i in 1 2 3; do
python tools/time_asm.py c2 30 tools/libmm_prev.so
python tools/time_asm.py c2 30
done
