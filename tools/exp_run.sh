# scratch driver for one gpurun call: 2 ranks on one GPU through gloo (host logic of the N > 1 bench path) on HEAD
FSTK_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-refit-none > gpurun_out/bench_g2b.log 2>&1; python - <<'PY'
import json
L=[x for x in open('gpurun_out/bench_g2b.log') if x.startswith('{')]
d=json.loads(L[-1]); r=d['refit']
print('n_gpus', d['n_gpus'], 'value', d['value'], 'refit', r['seconds'], r['samples_s'], 'steps', r['refine_steps'], 'lvl', r['gram_slices'], 'res', r['residual_after'])
PY
FSTK_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/bench_g2ref.log 2>&1; grep -c '"impl": "reference"' gpurun_out/bench_g2ref.log
