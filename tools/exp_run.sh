# scratch experiment driver (gpurun): solve variance with/without the cached Cholesky scratch
python -m pytest tests/test_gpu_gram.py -x -q -k cholesky > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
for v in "FSTK_CHOL_CACHE=1" "FSTK_CHOL_CACHE=0"; do echo "== $v"; env $v FSTK_DEBUG_TIMING=1 python tools/refit_var.py 8 2>&1 | grep -E "chol_crt|run " | sed 's/begin.*| dev//' | paste - - ; done > gpurun_out/exp_var.log 2>&1; cat gpurun_out/exp_var.log
