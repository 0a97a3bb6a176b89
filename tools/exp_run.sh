# scratch experiment driver (gpurun): the other BASELINE configs at full size (round-2 records)
python bench.py --config C3 --points 134217728 --steps 5 --warmup 3 --no-cpu --no-refit > gpurun_out/bench_c3.log 2>&1; tail -c 300 gpurun_out/bench_c3.log; echo
python bench.py --config C4 --points 268435456 --steps 3 --warmup 3 --no-cpu --no-refit-none > gpurun_out/bench_c4.log 2>&1; tail -c 300 gpurun_out/bench_c4.log; echo
python bench.py --config C1 --no-cpu > gpurun_out/bench_c1.log 2>&1; tail -c 300 gpurun_out/bench_c1.log; echo
