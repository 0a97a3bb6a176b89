# scratch experiment driver (gpurun): pair-pass sketch, prefetch placement
for m in 1 2 3 4; do FSTK_PP2_LD=$m FSTK_SKETCH_WARP2=1 timeout 300 python tools/sketch_time.py 3 > gpurun_out/sk_ld$m.log 2>&1; echo "LD=$m $(tail -n 1 gpurun_out/sk_ld$m.log)"; done
