# scratch experiment driver (gpurun): prepare phases after the prefetching sampler
python -m pytest tests/test_gpu_refit.py -x -q -k "sketch_rows or c1_refit or recovers or biased" > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 4 2>&1 | grep -E "^run|fstk prepare" | tail -16
