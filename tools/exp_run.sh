# scratch experiment driver (gpurun): parity subset + sketch timing A/B
K="sketch_rows or three_pass or c1_refit or 1m or columns"
python -m pytest tests/test_gpu_refit.py tests/test_gpu_columns.py -x -q -k "$K" > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
for r in 1 2; do for v in "FSTK_SKETCH_WLOCAL=1" "FSTK_SKETCH_WLOCAL=0"; do
  echo "== $v"; env $v python tools/sketch_time.py 3
done; done > gpurun_out/exp_time.log 2>&1
cat gpurun_out/exp_time.log
