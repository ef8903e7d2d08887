"""Steady-state time of the prep pass alone (cfg5): prepare_async + wait in a
loop, CUDA events around each call, for the sampled / full / no copy modes."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import bench
import paper_2010_07422_b200 as ir
from paper_2010_07422_b200 import gen, _capi
from paper_2010_07422_b200.solver import Context, _cover_sets
from paper_2010_07422_b200.sampling import pcg_words, draw_index_sets_from

cfgname = sys.argv[1] if len(sys.argv) > 1 else "cfg5"
n1, n2, r, al, dts, _ = bench.CONFIGS[cfgname]
D, linf, _ = gen.baseline_problem_device(n1, n2, r, al, bench.DATA_SEED, dtype=torch.float32 if dts == "f32" else torch.float64)
m = ir.sample_count(n1, r, 4.0)
cover = _cover_sets(ir.SolverConfig(rank=r, eps=bench.EPS, gamma=bench.GAMMA))
sets, _ = draw_index_sets_from(pcg_words(ir.RngSeed(1)), n1, n2, m, m, cover)
ctx = Context(0, _capi.F32 if dts == "f32" else _capi.F64, n1, n2, r, m, m, 100)
ctx.set_indices(sets)
st = torch.cuda.current_stream()
for mode in (2, 1, 0, 2):
    ts = []
    for i in range(6):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(st)
        ctx.prepare_async(D, mode, cover)
        b.record(st)
        ctx.prepare_wait()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    print(f"mode {mode}: " + " ".join(f"{t:.3f}" for t in ts) + " ms", flush=True)
