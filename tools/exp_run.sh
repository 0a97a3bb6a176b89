# scratch experiment driver (gpurun): rank-certificate chain enqueued by the side worker: parity + timing
timeout 1500 python -X faulthandler -m pytest tests/test_gpu_refit.py tests/test_gpu_gram.py tests/test_gpu_fullsize_refit.py tests/test_gpu_dist.py tests/test_gpu_cpp_shim.py -x -q > gpurun_out/exp_tests.log 2>&1; grep -v "^Extension" gpurun_out/exp_tests.log | tail -3
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 6 2>&1 | grep -E "^run|first solve" | tail -8
