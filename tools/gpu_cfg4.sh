# cfg4 batched path: parity tests, bench line with host-phase timings; prep tile-shape A/B at cfg5
set -x
timeout 600 python -m pytest tests/test_gpu_batched.py -x -q > gpurun_out/gputest_batched.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/gputest_batched.log
IRCUR_BATCH_PREP_PROF=1 timeout 300 python bench.py --config cfg4 --steps 10 --warmup 3 > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err; echo "cfg4 rc=$?"
python -c "import json;d=json.load(open('gpurun_out/bench_cfg4.json'));print('cfg4', d['value'],d['step_ms']);[print(p) for p in d['host_phases']]"
for sh in 1 2 1 2; do IRCUR_PREP_SHAPE=$sh timeout 300 python tools/prep_bench.py cfg5 2>&1 | sed "s/^/shape$sh /" | head -3; done
