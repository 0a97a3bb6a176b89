# scratch driver for one gpurun call (last use: the round's closing validation)
python -m pytest tests -m gpu -x -q > gpurun_out/gputests_h.log 2>&1; tail -n 2 gpurun_out/gputests_h.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_h.log 2>&1; tail -n 1 gpurun_out/smoke_h.log | cut -c1-220
python bench.py > gpurun_out/bench_h.log 2>&1; tail -c 200 gpurun_out/bench_h.log; echo
python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref_h.log 2>&1; tail -c 150 gpurun_out/bench_ref_h.log; echo
