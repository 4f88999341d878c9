mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err
for a in "--cfg B --r 12" "--cfg B --r 4" "--cfg B --r 1 --steps 4" "--cfg C --r 12" "--cfg C --r 4" "--cfg C --r 24" "--cfg C --r 1 --steps 4" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6" "--cfg E --r 4 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_a.jsonl 2>>gpurun_out/cfgs_a.err; done
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=30 > gpurun_out/pytest_a.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_a.log
