# scratch driver for one gpurun call: round-2 ncu capture of the contraction kernel
ncu --set full --clock-control none --import-source on -k regex:"contract_kernel" -s 2 -c 1 -o gpurun_out/contract_r02 python tools/prof_eval.py 22 3 C2 > gpurun_out/ncu_contract_r02.log 2>&1; tail -n 1 gpurun_out/ncu_contract_r02.log
