timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tf32" 2>&1 | tail -2
for i in 1 2 3; do
for p in 1 2; do
python tools/time_asm.py c2 30 tools/libmm_prev.so $p
python tools/time_asm.py c2 30 - $p
done
done
