nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_twophase.py -x -q > gpurun_out/pytest_tp.log 2>&1; echo pytest_tp $?
tail -3 gpurun_out/pytest_tp.log
timeout 600 python tools/time_twophase.py 6 > gpurun_out/twophase_s.log 2>&1; echo tp $?
grep "c4o2" gpurun_out/twophase_s.log
