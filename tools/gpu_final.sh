nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke $?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -3 gpurun_out/pytest_gpu.log
SECONDS=0; timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $? wall $SECONDS s
python -c "
import json; d=json.loads(open('gpurun_out/bench.json').readline()); r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'zf', r['incl_zero_fill']['frac'])
"
timeout 900 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo ref $?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-c4 > gpurun_out/b_ncu.log 2>&1; echo ncu1 $?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_asm_o1t" -c 1 -f -o gpurun_out/prof_c2 python tools/time_variant.py paper_2604_19286_b200/libmm.so c2 > /dev/null 2>&1; echo ncu2 $?
