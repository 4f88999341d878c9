mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "big or fullsize_one_step or bitwise" -x > gpurun_out/pytest_d.log 2>&1
echo "rc=$?" >> gpurun_out/pytest_d.log
for a in "--cfg B --r 12" "--cfg B --r 4" "--cfg C --r 12" "--cfg C --r 4" "--cfg C --r 1 --steps 4" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_d.jsonl 2>>gpurun_out/cfgs_d.err; done
