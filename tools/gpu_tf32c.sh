nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "tf32 or twophase or c4_full" > gpurun_out/pytest_tf32.log 2>&1; echo pytest_tf32 $?
tail -3 gpurun_out/pytest_tf32.log
timeout 600 python tools/time_twophase.py 6 > gpurun_out/twophase_c.log 2>&1; echo tp $?
grep "two_phase 0 \|two_phase 1 " gpurun_out/twophase_c.log
