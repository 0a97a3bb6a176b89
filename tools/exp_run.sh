# scratch experiment driver (gpurun): prepare phases with the two-thread sampler
FSTK_DEBUG_TIMING=1 python tools/refit_var.py 4 2>&1 | grep -E "^run|working subset|sketch plan" | tail -9
python -m pytest tests/test_gpu_refit.py -x -q -k "sketch_rows or c1_refit" 2>&1 | tail -n 1
