for cfg in "0 2" "1 2" "1e-2 2" "0 1" "1 1"; do set -- $cfg
  echo "JTHR=$1 SWEEPS=$2"; IRCUR_SVD_JTHR=$1 IRCUR_SVD_SWEEPS=$2 timeout 200 python tools/prof_run.py cfg5 --solves 2 2>&1 | grep -v Warn | grep -A2 "solve 1"
  IRCUR_SVD_JTHR=$1 IRCUR_SVD_SWEEPS=$2 timeout 200 python -c "
import paper_2010_07422_b200 as ir, bench, torch
from paper_2010_07422_b200 import gen
n1,n2,r,al,dts,_=bench.CONFIGS['cfg5']
D,linf,a=gen.baseline_problem_device(n1,n2,r,al,bench.DATA_SEED,dtype=torch.float32)
cfg=ir.SolverConfig(rank=r,eps=bench.EPS,zeta0=linf,gamma=bench.GAMMA,mode='resampled',max_iter=bench.MAX_ITER,seed=ir.RngSeed(bench.SOLVER_SEED))
res=ir.solve_device(D,cfg); print('iters',res.trace.iterations,'final_e',res.trace.errors[-1], 'e5', res.trace.errors[5])
" 2>&1 | tail -1
done
