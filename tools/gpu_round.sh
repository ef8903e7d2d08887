# Round-end evidence: default bench line, ncu launch list of the same command,
# the other configs' lines (profiles/ copies are made by hand from gpurun_out/).
mkdir -p gpurun_out
timeout 400 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; echo bench=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_final.csv \
  python bench.py --steps 1 --warmup 1 --e2e-steps 0 --no-cpu-baseline --no-clocks > gpurun_out/ncu_final.log 2>&1; echo ncu=$?
for c in ${CONFIGS:-cfg2 cfg3}; do
  timeout 400 python bench.py --config $c --no-cpu-baseline > gpurun_out/bench_final_$c.json 2> /dev/null; echo $c=$?
done
