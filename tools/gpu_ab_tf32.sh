timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tf32" 2>&1 | tail -3
for n in c2 c3; do
for p in 1 2; do
MM_TF32_REDS=1 python tools/time_asm.py $n 20 - $p
python tools/time_asm.py $n 20 - $p
done
done
