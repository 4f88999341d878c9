mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "big or fullsize_one_step or draw_ahead or bitwise" > gpurun_out/pytest_q.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_q.log
for a in "--cfg C --r 1 --burn 10" "--cfg C --r 4" "--cfg B --r 1 --burn 6 --steps 4" "--cfg B --r 4 --burn 6 --steps 4" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_q.jsonl 2>>gpurun_out/cfgs_q.err; done
