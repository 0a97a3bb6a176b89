# scratch experiment driver (gpurun): blocked int8 Cholesky level A/B (refit solve times)
for v in "FSTK_CHOL_CRT=7" "FSTK_CHOL_CRT=5" "FSTK_CHOL_CRT=6" "FSTK_CHOL_CRT=0"; do echo "== $v"; env $v python tools/refit_var.py 5 | sed 's/.*| dev//'; done > gpurun_out/exp_time.log 2>&1; cat gpurun_out/exp_time.log
