# scratch experiment driver (gpurun): full GPU tests + prepare timing
python -m pytest tests -m gpu -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
FSTK_DEBUG_TIMING=1 python tools/sketch_time.py 3 > gpurun_out/exp_prep.log 2>&1; tail -n 30 gpurun_out/exp_prep.log
