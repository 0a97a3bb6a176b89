# scratch driver for one gpurun call (last use: the round's closing validation of HEAD)
python -m pytest tests -m gpu -x -q > gpurun_out/gputests_i.log 2>&1; tail -n 2 gpurun_out/gputests_i.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_i.log 2>&1; tail -n 1 gpurun_out/smoke_i.log | cut -c1-220
python bench.py --steps 5 --warmup 3 > gpurun_out/bench_i.log 2>&1; tail -c 150 gpurun_out/bench_i.log; echo
