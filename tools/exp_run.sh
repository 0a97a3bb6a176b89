# scratch experiment driver (gpurun): eval parity + contraction L2 prefetch A/B
python -m pytest tests/test_gpu_eval.py -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
for r in 1 2; do
for v in "FSTK_CONTRACT_L2PF=1" "FSTK_CONTRACT_L2PF=0"; do
  echo "== $v"; env $v python tools/prof_eval.py 24 10 C2
done; done > gpurun_out/exp_time.log 2>&1
cat gpurun_out/exp_time.log
for v in "FSTK_CONTRACT_L2PF=1" "FSTK_CONTRACT_L2PF=0"; do env $v python bench.py --steps 20 --warmup 5 --no-cpu --no-refit > gpurun_out/b_$v.json 2>/dev/null; python -c "import json,sys; d=json.loads(open('gpurun_out/b_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['step_frac'])"; done
