# scratch experiment driver (gpurun): solve-stage variance inside the bench-like loop
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 8 > gpurun_out/exp_var.log 2>&1; grep -E "chol_crt|run " gpurun_out/exp_var.log | sed 's/begin.*| dev//'
