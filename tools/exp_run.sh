# scratch experiment driver (gpurun): new 2^20 parity tests + bench
python -m pytest tests/test_gpu_refit.py tests/test_gpu_columns.py -x -q -k "1m" > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
FSTK_SKETCH_WARP2=1 python -m pytest tests/test_gpu_refit.py tests/test_gpu_columns.py -x -q -k "1m" > gpurun_out/exp_tests2.log 2>&1; tail -n 2 gpurun_out/exp_tests2.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -n 2 gpurun_out/bench.err
