# scratch experiment driver (gpurun): level-3 Gram with 65,536-row segments (22 bits) against 32,768 (23 bits)
for seg in 32768 65536; do echo "seg=$seg"; FSTK_GRAM_SEG=$seg python tools/refit_var.py 4 2>&1 | grep -E "^run" | tail -3; done
FSTK_GRAM_SEG=65536 python -m pytest tests/test_gpu_gram.py tests/test_gpu_fullsize_refit.py -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
