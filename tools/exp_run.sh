# scratch experiment driver (gpurun): small-block cache; solve-time variance in the bench's refit loop
python -m pytest tests/test_gpu_refit.py tests/test_gpu_gram.py tests/test_gpu_rank.py tests/test_gpu_multi.py -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 3 gpurun_out/exp_tests.log
FSTK_DEBUG_TIMING=1 python bench.py --steps 3 --warmup 3 --no-cpu --refit-reps 6 > gpurun_out/bench_dbg.log 2> gpurun_out/bench_dbg.err; grep -E "fstk (alloc @factor|factor)" gpurun_out/bench_dbg.err | tail -30; python - <<'PY'
import json
l=[x for x in open('gpurun_out/bench_dbg.log') if x.startswith('{')][-1]
d=json.loads(l); print(d['refit']['samples_s'], [s['solve'] for s in d['refit']['sample_stages_s']], [s['prepare'] for s in d['refit']['sample_stages_s']]); print(d['refit_none']['samples_s'])
PY
