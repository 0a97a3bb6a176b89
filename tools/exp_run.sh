# scratch experiment driver (gpurun): parity subset + sketch timing variants
K="sketch_rows or three_pass or c1_refit or two_pass_1m"
FSTK_SKETCH_WARP2=1 python -m pytest tests/test_gpu_refit.py -x -q -k "$K" > gpurun_out/exp_tests2.log 2>&1; tail -n 2 gpurun_out/exp_tests2.log
for v in "FSTK_SKETCH_WARP2=1" "FSTK_SKETCH_WARP2=0"; do
  echo "== $v"; env $v python tools/sketch_time.py 3
done > gpurun_out/exp_time.log 2>&1
cat gpurun_out/exp_time.log
FSTK_SKETCH_WARP2=1 ncu --set full --clock-control none -k regex:"warp_pass2" -s 2 -c 1 -o gpurun_out/sketch_v3b python tools/sketch_time.py 1 > gpurun_out/ncu_sketch.log 2>&1; tail -n 1 gpurun_out/ncu_sketch.log
