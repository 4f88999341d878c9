mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "lasso or nmf or enet or codes_variants or cfgB or cfgD or cfgE" > gpurun_out/pytest_j.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_j.log
for a in "--cfg B --r 12" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_j.jsonl 2>>gpurun_out/cfgs_j.err; done
