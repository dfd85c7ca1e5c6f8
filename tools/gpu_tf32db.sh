nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "tf32 or twophase" > gpurun_out/pytest_tf32.log 2>&1; echo pytest_tf32 $?
tail -4 gpurun_out/pytest_tf32.log
timeout 600 python tools/time_twophase.py 6 c2 > gpurun_out/twophase_db.log 2>&1; echo tp $?
grep "two_phase 0 \|two_phase 1 \|two_phase 2 \|two_phase 9 \|two_phase 10 " gpurun_out/twophase_db.log
