set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest.log
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err; echo "bench rc=$?"
cat gpurun_out/bench_cfg5.json | head -c 1500
timeout 300 python bench.py --config cfg4 --steps 5 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
head -c 800 gpurun_out/bench_cfg4.json
