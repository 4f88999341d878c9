mkdir -p gpurun_out
for c in 1 2 4 8 16; do timeout 300 python tests/tools/run_cfg.py --cfg C --r 12 --copies $c >> gpurun_out/copies.jsonl 2>>gpurun_out/copies.err; done
timeout 300 python tests/tools/run_cfg.py --cfg B --r 12 >> gpurun_out/cfgB.jsonl 2>>gpurun_out/cfgB.err
ncu --set full --clock-control none --import-source on -k regex:k_bcd_big -s 5 -c 1 -o gpurun_out/ncu_big -f python tests/tools/run_cfg.py --cfg B --r 12 --steps 2 --burn 6 > gpurun_out/ncu_big.log 2>&1
