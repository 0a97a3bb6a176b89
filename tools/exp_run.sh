# scratch experiment driver (gpurun): level-3 Gram default + extrapolated stop: parity suite, C4/C5 refits
python -m pytest tests -m gpu -x -q > gpurun_out/gputests_c.log 2>&1; tail -n 3 gpurun_out/gputests_c.log
python bench.py --config C4 --no-cpu --no-refit-none --steps 3 --warmup 3 > gpurun_out/bench_c4b.log 2>&1; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_c4b.log') if x.startswith('{')][-1]
d=json.loads(l)
r=d['refit']; print('C4', r['seconds'], r['samples_s'], 'hot', r['hot_path_seconds'], 'steps', r['refine_steps'], 'lvl', r['gram_slices'], r['sample_stages_s'][0], 'res', r['residual_after'])
PY
python bench.py --config C5 --no-cpu --no-refit-none --steps 3 --warmup 3 > gpurun_out/bench_c5b.log 2>&1; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_c5b.log') if x.startswith('{')][-1]
d=json.loads(l)
r=d['refit']; print('C5', r['seconds'], r['samples_s'], 'steps', r['refine_steps'], 'lvl', r['gram_slices']); print(d.get('refit_fields'))
PY
