mkdir -p gpurun_out
for a in "--cfg C --r 1 --burn 10" "--cfg C --r 4" "--cfg B --r 1 --burn 6 --steps 4" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_p.jsonl 2>>gpurun_out/cfgs_p.err; done
