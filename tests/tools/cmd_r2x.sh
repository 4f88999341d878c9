mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_x.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_x.log
timeout 2700 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/pytest_x.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_x.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_x.json 2> gpurun_out/bench_x.err
echo "bench rc=$?" >> gpurun_out/bench_x.err
