# scratch experiment driver (gpurun): refinement steps of the transform="none" refit by Gram level
for l in 4 3 2; do echo "level $l"; FSTK_GRAM_SLICES=$l python tools/refine_time.py 1 none 2>&1 | grep -E "steps|rror" | cut -c1-220; done
