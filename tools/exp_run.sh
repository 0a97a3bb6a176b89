# scratch experiment driver (gpurun): parity + sketch timing A/B (pass-1 register twiddles, 8 warps)
K="sketch_rows or three_pass or 1m"
FSTK_SKETCH_WARP=8 FSTK_SKETCH_W1RT=1 python -m pytest tests/test_gpu_refit.py -x -q -k "$K" > gpurun_out/exp_tests.log 2>&1; tail -n 1 gpurun_out/exp_tests.log
for r in 1 2; do for v in "FSTK_SKETCH_WARP=8 FSTK_SKETCH_W1RT=1" "FSTK_SKETCH_WARP=12" "FSTK_SKETCH_WARP=8"; do echo "== $v"; env $v python tools/sketch_time.py 3; done; done > gpurun_out/exp_time.log 2>&1; cat gpurun_out/exp_time.log
