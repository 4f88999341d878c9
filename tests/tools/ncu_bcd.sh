#!/bin/bash
# ncu capture of one BCD launch at cfgC r=12 (steady state), source-level
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:k_bcd_newton -s 40 -c 1 \
    -o gpurun_out/ncu_bcd -f python bench.py --steps 3 --warmup 3 --burn-in 40 --no-sweep --no-e2e --no-cpu \
    > gpurun_out/ncu_bcd.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_bcd.log
