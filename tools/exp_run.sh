# scratch experiment driver (gpurun): bench refit samples with stage breakdown
python bench.py --steps 20 --warmup 5 --no-cpu --no-refit-none --refit-reps 5 > gpurun_out/b.json 2>/dev/null
python -c "
import json; d=json.loads(open('gpurun_out/b.json').read().strip().splitlines()[-1]); r=d['refit']; print(r['seconds'], r['samples_s'])
for x in r['sample_stages_s']: print(x)"
