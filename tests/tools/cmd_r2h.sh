mkdir -p gpurun_out
timeout 600 python tests/tools/cap_repro.py --cfg E --r 24 --steps 12 > gpurun_out/cap_h.jsonl 2>gpurun_out/cap_h.err
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "one_step_parity or draw_ahead or project" > gpurun_out/pytest_h.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_h.log
