# Every bench config with the overlapped loop (default) and the sequential
# loop (IRCUR_OVERLAP=0), same box: value and e2e per line.
mkdir -p gpurun_out
for c in cfg2 cfg3 video_mall video_restaurant cfg4; do
  for ov in 1 0; do
    IRCUR_OVERLAP=$ov timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/sweep_${c}_ov$ov.json 2> gpurun_out/sweep_${c}_ov$ov.err
    python -c "import json,sys; d=json.load(open('gpurun_out/sweep_${c}_ov$ov.json')); print('$c', 'overlap=$ov', round(d['value']*1e3,3), 'ms', 'e2e', round(d['e2e']['value'],4), d['breakdown_ms_per_solve'].get('loop') if 'breakdown_ms_per_solve' in d else '')" 2>&1 | tail -1
  done
done
