mkdir -p gpurun_out
timeout 600 python tests/tools/cap_repro.py --cfg E --r 24 --steps 10 > gpurun_out/cap_e.jsonl 2>gpurun_out/cap_e.err
timeout 300 python tests/tools/cap_repro.py --cfg B --r 12 --steps 6 >> gpurun_out/cap_e.jsonl 2>>gpurun_out/cap_e.err
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "big or bitwise or fullsize_one_step or k256" > gpurun_out/pytest_e.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_e.log
