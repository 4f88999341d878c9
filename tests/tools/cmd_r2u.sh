mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_u.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_u.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_u.json 2> gpurun_out/bench_u.err
echo "bench rc=$?" >> gpurun_out/bench_u.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_ref_u.json 2> gpurun_out/bench_ref_u.err
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/pytest_u.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_u.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches_u.csv python bench.py --steps 5 --warmup 3 --burn-in 30 --no-sweep --no-e2e --no-cpu > gpurun_out/ncu_launch_u.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_launch_u.log
bash tests/tools/ncu_bcd.sh
bash tests/tools/ncu_others.sh
