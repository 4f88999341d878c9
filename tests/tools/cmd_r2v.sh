mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "phase_clocks or full_size_fmri_step or cfgA" > gpurun_out/pytest_v.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_v.log
