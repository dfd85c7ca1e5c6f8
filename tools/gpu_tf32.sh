timeout 600 python -m pytest tests -m gpu -x -q -k "tf32" > gpurun_out/pytest_tf32.log 2>&1; echo pytest $?; tail -15 gpurun_out/pytest_tf32.log
timeout 300 python tools/time_tf32.py c2
timeout 300 python tools/time_tf32.py c3
