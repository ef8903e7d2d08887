set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests_k.log 2>&1; tail -3 gpurun_out/gpu_tests_k.log
timeout 300 python bench.py > gpurun_out/bench_k.json 2> gpurun_out/bench_k.err; tail -c 600 gpurun_out/bench_k.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r1k.csv python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks > gpurun_out/ncu_k.log 2>&1; echo ncu1=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sampled_staged -s 20 -c 1 -f -o gpurun_out/sampled_r1k python tools/prof_run.py cfg5 --solves 1 > gpurun_out/ncu_s.log 2>&1; echo ncu2=$?
timeout 600 ncu --set full --clock-control none --import-source on -k regex:strips3 -s 20 -c 1 -f -o gpurun_out/strips3_r1k python tools/prof_run.py cfg5 --solves 1 > gpurun_out/ncu_t.log 2>&1; echo ncu3=$?
