mkdir -p gpurun_out
for a in "--group 1" "--group 2" "--group 4" "--group 2 --r 24" "--group 1 --r 24" "--group 4 --r 24"; do timeout 300 python tests/tools/run_cfg.py --cfg C --burn 60 $a >> gpurun_out/cfgs_k.jsonl 2>>gpurun_out/cfgs_k.err; done
