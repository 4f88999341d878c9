mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "(one_step_parity and (fmri or cfgA or nmf_small or full_mode)) or fmri_support or (contract_variants and tc) or (bbar_variants and tc) or bitwise" > gpurun_out/pytest_t.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_t.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_t.json 2> gpurun_out/bench_t.err
echo "bench rc=$?" >> gpurun_out/bench_t.err
