mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_shard.py -m gpu -q -p no:cacheprovider > gpurun_out/pytest_m.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m.log
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 5 --warmup 3 --burn-in 10 --no-sweep --no-cpu > gpurun_out/bench_2rank_m.json 2> gpurun_out/bench_2rank_m.err
echo "bench rc=$?" >> gpurun_out/bench_2rank_m.err
for a in "--cfg B --r 12" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_m.jsonl 2>>gpurun_out/cfgs_m.err; done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "lasso or nmf or enet or codes_variants or cfgB or cfgD or cfgE or estimator" > gpurun_out/pytest_m2.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_m2.log
