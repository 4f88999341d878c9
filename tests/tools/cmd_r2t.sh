mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -x -k "one_step_parity and (fmri or cfgA or nmf_small)" > gpurun_out/pytest_t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_t.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
echo "bench rc=$?" >> gpurun_out/bench_t.err
