# scratch experiment driver (gpurun): refit tests + prepare timing
python -m pytest tests/test_gpu_refit.py tests/test_gpu_threads.py tests/test_gpu_dist.py -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 4 > gpurun_out/exp_prep.log 2>&1; grep -E "compact|working|run " gpurun_out/exp_prep.log | sed 's/gram 1.*//'
