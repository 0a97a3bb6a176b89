# scratch experiment driver (gpurun): next segment's residues on a side stream beside the SYRKs
python -m pytest tests/test_gpu_gram.py tests/test_gpu_refit.py tests/test_gpu_fullsize_refit.py tests/test_gpu_multi.py tests/test_gpu_scale.py -x -q 2>&1 | tail -n 1
for o in 0 1; do echo "overlap=$o"; FSTK_GRAM_OVERLAP=$o python tools/refit_var.py 5 2>&1 | grep -E "^run" | tail -3; done
