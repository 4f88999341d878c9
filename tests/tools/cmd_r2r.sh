mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_r.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_r.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r.json 2> gpurun_out/bench_r.err
echo "bench rc=$?" >> gpurun_out/bench_r.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_r.json 2> gpurun_out/bench_ref_r.err
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_r.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_r.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_r.csv python bench.py --steps 5 --warmup 3 --burn-in 30 --no-sweep --no-e2e --no-cpu > gpurun_out/ncu_launch_r.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_r.log
bash tests/tools/ncu_bcd.sh
bash tests/tools/ncu_others.sh
