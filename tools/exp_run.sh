# scratch experiment driver (gpurun): final records: default bench, reference arm, launch list
python bench.py > gpurun_out/bench_d.log 2>&1; tail -c 300 gpurun_out/bench_d.log; echo
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_d.log 2>&1; tail -c 200 gpurun_out/bench_ref_d.log; echo
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_bench_r02_v2.csv python bench.py --steps 2 --warmup 3 --no-cpu --no-refit-none --refit-warmup 0 --refit-reps 1 > gpurun_out/ncu_d.log 2>&1; tail -n 1 gpurun_out/ncu_d.log | cut -c1-200
