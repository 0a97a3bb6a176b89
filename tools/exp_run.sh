# scratch experiment driver (gpurun): Cholesky lookahead with the next panel enqueued from inside the update
python -m pytest tests/test_gpu_gram.py tests/test_gpu_refit.py -x -q 2>&1 | tail -n 1
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 6 2>&1 | grep -E "^run|chol_crt" | tail -10
python tools/chol_time.py 4 2>&1 | grep "slices=5"
