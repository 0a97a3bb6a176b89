# scratch driver for one gpurun call (last use: HEAD sanity after the debug instrumentation)
python -m pytest tests/test_gpu_gram.py tests/test_gpu_refit.py tests/test_gpu_rank.py -x -q 2>&1 | tail -n 1
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -n 1 | cut -c1-160
python tools/refit_var.py 4 2>&1 | grep -E "^run" | tail -3
