# scratch experiment driver (gpurun): 2 ranks on one GPU through gloo (host logic of the N > 1 bench path)
FSTK_BENCH_BACKEND=gloo timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --no-refit-none > gpurun_out/bench_g2.log 2>&1; tail -c 1500 gpurun_out/bench_g2.log
