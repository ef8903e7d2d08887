# prep pass time per tile shape / grid (tools/prep_bench.py), cfg5
for sh in 0 1; do echo "IRCUR_PREP_SHAPE=$sh"; IRCUR_PREP_SHAPE=$sh timeout 300 python tools/prep_bench.py 2>&1 | grep "mode 2" | tail -1; done
