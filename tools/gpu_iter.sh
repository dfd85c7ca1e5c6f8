timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest $?
tail -4 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 100 --no-tf32 --no-e2e --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench $?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench.json').read().strip().splitlines()[-1])
b=d['breakdown']; print('c2 step', d['ms_per_step'], 'sort', b['sort_ms'], 'asm', b['assemble_ms'], 'asm alone', b['assemble_alone_ms'])
o=d.get('order2',{}); print('c3 step', o.get('ms_per_step'), 'sort', o.get('sort_ms'), 'asm', o.get('assemble_ms'))
PY
tail -3 gpurun_out/bench.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-tf32 > /dev/null 2>&1; echo ncu $?
