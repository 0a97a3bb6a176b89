# scratch driver for one gpurun call (parity subset + timings of whatever is being tried);
# its contents are whatever the latest experiment was.  Closing state of round 2:
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; tail -n 2 gpurun_out/gputests.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1
python bench.py > gpurun_out/bench.log 2>&1; tail -c 300 gpurun_out/bench.log
