nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "tf32 or twophase or zeroing" > gpurun_out/pytest_tf32.log 2>&1; echo pytest_tf32 $?
tail -3 gpurun_out/pytest_tf32.log
timeout 600 python tools/time_twophase.py 6 c2 > gpurun_out/twophase_d.log 2>&1; echo tp $?
grep "two_phase 0 " gpurun_out/twophase_d.log
SECONDS=0; timeout 900 python bench.py --no-cpu-baseline > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err; echo bench $? $SECONDS
python -c "
import json; d=json.loads(open('gpurun_out/bench_d.json').readline()); r=d['roofline']
print('value', d['value'], 'ms', d['ms_per_step'], 'kernel_ms', r['kernel_ms'], 'frac', r['frac'], 'zf', r['incl_zero_fill'])
print({k:(v['assemble_ms'], v['roofline']['frac']) for k,v in d['tf32'].items()})
"
