nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
for a in "" "--no-zero-overlap" "" "--no-zero-overlap"; do
timeout 600 python bench.py --no-cpu-baseline --no-e2e --no-c4 --no-weak --no-tf32 --no-order2 $a > gpurun_out/zo.json 2> gpurun_out/zo.err; echo "bench[$a] $?"
python -c "
import json; d=json.loads(open('gpurun_out/zo.json').readline()); b=d['breakdown']
print(round(d['value']), round(d['ms_per_step'],4), b['step_schedule'][:30], 'asm', round(b['assemble_ms'],4), 'sort', round(b['sort_async_ms'],4), 'frac', round(d['roofline']['frac'],4), round(d['roofline']['incl_zero_fill']['frac'],4))
"
done
