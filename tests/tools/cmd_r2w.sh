mkdir -p gpurun_out
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 10 --warmup 3 --no-sweep --no-cpu > gpurun_out/bench_2rank_w.json 2> gpurun_out/bench_2rank_w.err
echo "bench rc=$?" >> gpurun_out/bench_2rank_w.err
