mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "unbiased or (one_step_parity and (newton or big)) or draw_ahead" > gpurun_out/pytest_c.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_c.log
timeout 400 python tests/tools/cap_repro.py --cfg E --r 24 --steps 12 > gpurun_out/cap_c.jsonl 2>gpurun_out/cap_c.err
for a in "--cfg B --r 12" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6" "--cfg E --r 24 --steps 3 --burn 10"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_c.jsonl 2>>gpurun_out/cfgs_c.err; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_c.json 2> gpurun_out/bench_c.err
echo "bench rc=$?" >> gpurun_out/bench_c.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/ncu_launch_c.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_c.log
bash tests/tools/ncu_bcd.sh
