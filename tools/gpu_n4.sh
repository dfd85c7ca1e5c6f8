#!/bin/bash
timeout 300 python -m pytest tests/test_gpu_next4.py -q -x > gpurun_out/n4_pytest.log 2>&1; echo "next4 tests rc $?"; tail -1 gpurun_out/n4_pytest.log
for i in 1 2; do echo "next4: $(timeout 300 python tools/time_next4.py - 2>&1 | tail -3 | tr '\n' ' ')"; done
