#!/bin/bash
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_moments|k_gather" -s 3 -c 3 -f -o gpurun_out/n4 python tools/time_next4.py - > gpurun_out/n4_ncu.log 2>&1; echo "ncu rc $?"
