# scratch experiment driver (gpurun): parity subset + sketch timing
K="sketch_rows or three_pass or c1_refit or 1m"
python -m pytest tests/test_gpu_refit.py tests/test_gpu_columns.py -x -q -k "$K" > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
python tools/sketch_time.py 5 > gpurun_out/exp_time.log 2>&1; cat gpurun_out/exp_time.log
ncu --set full --clock-control none -k regex:"warp_pass1" -s 2 -c 1 -o gpurun_out/wp1r python tools/sketch_time.py 1 > /dev/null 2>&1
