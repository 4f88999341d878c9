mkdir -p gpurun_out
timeout 400 python tests/tools/cap_repro.py --cfg E --r 24 --steps 12 > gpurun_out/cap_d.jsonl 2>gpurun_out/cap_d.err
for a in "--cfg B --r 12" "--cfg D --r 8" "--cfg E --r 12 --steps 3 --burn 6"; do timeout 300 python tests/tools/run_cfg.py $a >> gpurun_out/cfgs_d.jsonl 2>>gpurun_out/cfgs_d.err; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -q -p no:cacheprovider -x -k "lasso or nmf or enet or codes_variants or fullsize_one_step" > gpurun_out/pytest_d.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_d.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_d.json 2> gpurun_out/bench_d.err
echo "bench rc=$?" >> gpurun_out/bench_d.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_d.csv python bench.py --steps 5 --warmup 3 --no-sweep --no-e2e --no-cpu > gpurun_out/ncu_launch_d.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_d.log
bash tests/tools/ncu_bcd.sh
