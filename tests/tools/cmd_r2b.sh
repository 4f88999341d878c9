mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -p no:cacheprovider -k "unbiased or draw_ahead or (one_step_parity and (newton or big))" > gpurun_out/pytest_b.log 2>&1
echo "pytest rc=$?" >> gpurun_out/pytest_b.log
for a in "--cfg E --r 24 --steps 16" "--cfg B --r 12 --steps 16" "--cfg B --r 1 --steps 12" "--cfg D --r 8 --steps 16"; do timeout 400 python tests/tools/cap_repro.py $a >> gpurun_out/cap_b.jsonl 2>>gpurun_out/cap_b.err; done
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_b.json 2> gpurun_out/bench_b.err
echo "bench rc=$?" >> gpurun_out/bench_b.err
SAN_STEPS=2 timeout 1200 compute-sanitizer --tool racecheck --print-limit 50 python tests/tools/sanitize_run.py > gpurun_out/san_race.log 2>&1
echo "rc=$?" >> gpurun_out/san_race.log
SAN_STEPS=2 timeout 900 compute-sanitizer --tool synccheck --print-limit 50 python tests/tools/sanitize_run.py > gpurun_out/san_sync.log 2>&1
echo "rc=$?" >> gpurun_out/san_sync.log
SAN_STEPS=2 timeout 900 compute-sanitizer --tool memcheck --print-limit 50 python tests/tools/sanitize_run.py > gpurun_out/san_mem.log 2>&1
echo "rc=$?" >> gpurun_out/san_mem.log
