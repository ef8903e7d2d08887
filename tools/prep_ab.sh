# same-box A/B of the prep pass variants (tools/prep_bench.py, cfg5)
for rep in 1 2; do for nm in 0 1; do echo "NANMAX=$nm"; IRCUR_PREP_NANMAX=$nm timeout 300 python tools/prep_bench.py 2>&1 | grep "mode 2" | tail -1; done; done
