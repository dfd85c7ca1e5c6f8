timeout 600 python -m pytest tests -m gpu -x -q -k "uniform or clustered or lattice or c1 or slab or accumulate or species or spacing or empty or special" > gpurun_out/pytest_s.log 2>&1; echo pytest $?; tail -5 gpurun_out/pytest_s.log
timeout 300 python tools/time_c4.py 1 5
timeout 300 python tools/time_c4.py 2 5
