nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 python tools/time_twophase.py 6 > gpurun_out/twophase.log 2>&1; echo tp $?
cat gpurun_out/twophase.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_nodesum|k_asm_tf32" -c 4 -f -o gpurun_out/prof_tp python tools/prof_twophase.py 1 > gpurun_out/prof_tp.log 2>&1; echo ncu $?
tail -3 gpurun_out/prof_tp.log
