mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "sweep" > gpurun_out/pytest_i.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i.log
for a in "--codes-kernel sweep" "--codes-kernel ridge" "--codes-kernel sweep"; do timeout 300 python tests/tools/run_cfg.py --cfg C --r 12 --burn 60 $a >> gpurun_out/cfgs_i.jsonl 2>>gpurun_out/cfgs_i.err; done
timeout 900 python -m pytest tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "codes_variants and sweep" >> gpurun_out/pytest_i.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_i.log
