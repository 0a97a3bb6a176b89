# scratch experiment driver (gpurun): Gram tests + fold profile + Gram time
python -m pytest tests/test_gpu_gram.py tests/test_gpu_refit.py -x -q > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
python tools/prof_gram.py 4 > gpurun_out/pg.log 2>&1; python tools/prof_gram.py 4 >> gpurun_out/pg.log 2>&1; cat gpurun_out/pg.log
ncu --set full --clock-control none -k regex:"crt_fold" -s 20 -c 1 -o gpurun_out/fold2 python tools/prof_gram.py 4 > /dev/null 2>&1
