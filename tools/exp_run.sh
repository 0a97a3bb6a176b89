# scratch experiment driver (gpurun): full GPU suite + bench + reference arm + launch list
python -m pytest tests -m gpu -x -q > gpurun_out/gputests_b.log 2>&1; tail -n 3 gpurun_out/gputests_b.log
python bench.py > gpurun_out/bench_b.log 2>&1; tail -c 600 gpurun_out/bench_b.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_b.log 2>&1; tail -n 2 gpurun_out/smoke_b.log
