mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "big or masked_api or fullsize_one_step or draw_ahead" > gpurun_out/pytest_o.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_o.log
for a in "--cfg C --r 1 --burn 10" "--cfg C --r 4" "--cfg C --r 12" "--cfg B --r 12" "--cfg B --r 1 --burn 6 --steps 4"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_o.jsonl 2>>gpurun_out/cfgs_o.err; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_o.json 2> gpurun_out/bench_o.err
echo "bench rc=$?" >> gpurun_out/bench_o.err
