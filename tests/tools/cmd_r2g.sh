mkdir -p gpurun_out
timeout 600 python tests/tools/cap_repro.py --cfg E --r 24 --steps 5 > gpurun_out/cap_g.jsonl 2>gpurun_out/cap_g.err
timeout 300 python tests/tools/run_cfg.py --cfg C --r 12 --burn 60 > gpurun_out/cfgs_g.jsonl 2>gpurun_out/cfgs_g.err
