mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "one_step or fmri_support or bbar_variants or contract_variants or bitwise or trajectory_small or estimator" > gpurun_out/pytest_s.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_s.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_s.json 2> gpurun_out/bench_s.err
echo "bench rc=$?" >> gpurun_out/bench_s.err
