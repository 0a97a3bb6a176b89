# scratch experiment driver (gpurun): pair-pass sketch with 6 pairs (12 warps), rotations from L2
FSTK_SKETCH_WARP2=1 timeout 600 python -m pytest tests/test_gpu_refit.py -x -q -k "two_pass_1m" > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
FSTK_SKETCH_WARP2=1 timeout 300 python tools/sketch_time.py 3 2>&1 | tail -n 2
FSTK_SKETCH_WARP2=0 timeout 300 python tools/sketch_time.py 3 2>&1 | tail -n 1
