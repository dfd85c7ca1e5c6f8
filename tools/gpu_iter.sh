timeout 600 python -m pytest tests -m gpu -x -q -k "sort or c1 or parity_uniform or clustered or errors or empty or slab or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -15 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --no-tf32 --no-e2e --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
tail -c 1500 gpurun_out/bench.json; tail -5 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches_sort.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tf32 --no-order2 > /dev/null 2>&1; echo ncu $?
