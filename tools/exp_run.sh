# scratch driver for one gpurun call: level rule by oversampling: tests + C1/C2 refits
python -m pytest tests/test_gpu_gram.py tests/test_gpu_refit.py tests/test_gpu_rank.py tests/test_gpu_multi.py tests/test_gpu_dist.py -x -q 2>&1 | tail -n 1
python bench.py --config C1 --no-cpu --steps 3 --warmup 3 > gpurun_out/bench_c1c.log 2>&1; python - <<'PY'
import json
d=json.loads([x for x in open('gpurun_out/bench_c1c.log') if x.startswith('{')][-1])
r=d['refit']; print('C1:', r['seconds'], r['samples_s'], 'steps', r['refine_steps'], 'used', r['gram_slices'])
PY
python tools/refit_var.py 3 2>&1 | grep -E "^run" | tail -2
