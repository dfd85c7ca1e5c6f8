# Round measurement: smoke, GPU tests, full bench, launch list, ncu full captures of the hot kernels.
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $? wall $SECONDS s
tail -3 gpurun_out/bench.err
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4 > gpurun_out/b_ncu.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_asm_o1t" -c 1 -f -o gpurun_out/prof_c2 python tools/time_variant.py paper_2604_19286_b200/libmm.so c2 > /dev/null 2>&1; echo ncu2 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_key|k_place|k_fix_warp|k_scatter" -c 4 -f -o gpurun_out/prof_sort python tools/time_sort.py c2 2 > /dev/null 2>&1; echo ncu2b $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_asm_o2t" -c 1 -f -o gpurun_out/prof_c3 python tools/time_variant.py paper_2604_19286_b200/libmm.so c3 > /dev/null 2>&1; echo ncu3 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_asm_tf32" -c 1 -f -o gpurun_out/prof_tf32 python tools/time_tf32.py c2 > /dev/null 2>&1; echo ncu4 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_asm_pps" -c 1 -f -o gpurun_out/prof_c4o2 python tools/time_c4.py 2 1 > /dev/null 2>&1; echo ncu5 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_apply" -c 1 -f -o gpurun_out/prof_apply python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-e2e --no-tf32 --no-order2 --no-c4 > /dev/null 2>&1; echo ncu6 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_moments|k_gather" -c 2 -f -o gpurun_out/prof_next4 python tools/time_next4.py > /dev/null 2>&1; echo ncu7 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_scatter0|k_fixrec_warp" -c 2 -f -o gpurun_out/prof_recfirst python tools/time_sort_big.py 1 > /dev/null 2>&1; echo ncu8 $?
