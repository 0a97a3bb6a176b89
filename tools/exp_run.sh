# scratch driver for one gpurun call: Cholesky factor outliers (per-panel device and host times)
FSTK_DEBUG_TIMING=1 python bench.py --steps 3 --warmup 3 --no-cpu --no-refit-none --refit-reps 12 > gpurun_out/bench_j.log 2> gpurun_out/bench_j.err
grep -E "chol_crt|chol panels" gpurun_out/bench_j.err | tail -30
