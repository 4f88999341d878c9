mkdir -p gpurun_out
for c in 1 2 4 8; do timeout 300 python tests/tools/run_cfg.py --cfg C --r 12 --copies $c --burn 60 >> gpurun_out/copies2.jsonl 2>>gpurun_out/copies2.err; done
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "newton or big" -x > gpurun_out/pytest_c.log 2>&1
