set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -c 3000 gpurun_out/bench.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tf32 > gpurun_out/b_ncu.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_asm -c 2 -f -o gpurun_out/asm_full python bench.py --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-tf32 > gpurun_out/b_ncu2.log 2>&1; echo ncu2 $?
