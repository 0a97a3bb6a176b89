# scratch experiment driver (gpurun): parity subset + sketch timing
K="sketch_rows or three_pass or c1_refit or two_pass_1m or sharded or columns"
python -m pytest tests/test_gpu_refit.py tests/test_gpu_columns.py -x -q -k "$K" > gpurun_out/exp_tests.log 2>&1; tail -n 2 gpurun_out/exp_tests.log
python tools/sketch_time.py 4 > gpurun_out/exp_time.log 2>&1
cat gpurun_out/exp_time.log
