mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -k "newton or draw_ahead or fmri or bitwise or empty or trajectory_objective" > gpurun_out/pytest_f.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_f.log
timeout 300 python tests/tools/run_cfg.py --cfg C --r 12 --burn 60 > gpurun_out/cfgs_f.jsonl 2>gpurun_out/cfgs_f.err
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_f.json 2> gpurun_out/bench_f.err
echo "bench rc=$?" >> gpurun_out/bench_f.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_f.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/ncu_launch_f.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_f.log
