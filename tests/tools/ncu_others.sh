#!/bin/bash
# ncu capture (full set, source) of the contraction, ridge-codes and B-bar kernels at cfgC r=12
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"k_contract_tc|k_bbar_tc|k_ridge_codes" -s 60 -c 3 \
    -o gpurun_out/ncu_others -f python tests/tools/run_cfg.py --cfg C --r 12 --steps 3 --burn 20 \
    > gpurun_out/ncu_others.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_others.log
