timeout 600 python -m pytest tests -m gpu -x -q -k "apply" 2>&1 | tail -3
timeout 600 python bench.py --steps 50 --no-tf32 --no-e2e --no-cpu-baseline --no-c4 > gpurun_out/bench_ap.json 2> gpurun_out/bench_ap.err; echo bench $?; tail -3 gpurun_out/bench_ap.err
python -c "
import json; d=json.loads(open('gpurun_out/bench_ap.json').read().strip().splitlines()[-1]); print(d.get('apply')); print(d['order2'].get('apply'))"
