python -m pytest tests -m gpu -x -q > gpurun_out/gputests_a.log 2>&1; tail -n 3 gpurun_out/gputests_a.log
python bench.py > gpurun_out/bench_a.log 2>&1; tail -n 2 gpurun_out/bench_a.log
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_a.log 2>&1; tail -n 1 gpurun_out/bench_ref_a.log
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench_r02.csv python bench.py --steps 2 --warmup 1 > gpurun_out/ncu_a.log 2>&1; tail -n 2 gpurun_out/ncu_a.log
