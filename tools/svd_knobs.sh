for ex in -1 4 2; do for sw in 2 1; do
  echo "extra=$ex sweeps=$sw"; IRCUR_SVD_EXTRA=$ex IRCUR_SVD_SWEEPS=$sw timeout 200 python tools/prof_run.py cfg5 --solves 2 2>&1 | grep -v Warn | sed -n 4,6p
done; done
for ex in -1 4; do IRCUR_SVD_EXTRA=$ex IRCUR_SVD_SWEEPS=1 timeout 200 python tools/prof_run.py cfg2 --solves 2 2>&1 | grep -v Warn | sed -n 4,4p; done
