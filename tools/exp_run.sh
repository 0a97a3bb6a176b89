# scratch experiment driver (gpurun): bench refit with the Cholesky lookahead on/off
for la in 0 1; do FSTK_CHOL_LOOKAHEAD=$la FSTK_DEBUG_TIMING=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-refit-none --refit-reps 6 > gpurun_out/bench_la$la.log 2> gpurun_out/bench_la$la.err; grep -E "chol_crt" gpurun_out/bench_la$la.err | tr '\n' ' '; python - <<PY
import json
l=[x for x in open('gpurun_out/bench_la$la.log') if x.startswith('{')][-1]
d=json.loads(l); print('\nlookahead=$la', d['refit']['samples_s'], [s['solve'] for s in d['refit']['sample_stages_s']])
PY
done
