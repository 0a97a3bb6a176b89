# scratch experiment driver (gpurun): single-CTA triangular block solves against cuBLAS TRSV/TRSM
python -m pytest tests/test_gpu_rank.py tests/test_gpu_refit.py tests/test_gpu_gram.py tests/test_gpu_multi.py tests/test_gpu_fullsize_refit.py -x -q 2>&1 | tail -n 1
for c in 0 1; do echo "custom=$c"; FSTK_TRI_CUSTOM=$c python tools/refit_var.py 5 2>&1 | grep -E "^run" | tail -3; FSTK_TRI_CUSTOM=$c python tools/refine_time.py 1 2>&1 | grep -E "rep 0" | cut -c1-260; done
