import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, numpy as np, qtgen, paper_1912_10024_b200 as qt
from tests.helpers import MICROS, micro, inputs
cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 0
which = sys.argv[2] if len(sys.argv) > 2 else "both"
p = micro(**MICROS[cfg])
inp = inputs(p, seed=300 + cfg)
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
sh = p.shapes()
o = {k: torch.empty(sh["G" if k[0] == "S" else "D"], dtype=torch.complex128, device="cuda") for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
plan = qt.Plan(p); print(plan.info(), flush=True)
if which in ("both", "sigma"):
    plan.sigma(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], o["S_less"], o["S_gtr"]); torch.cuda.synchronize(); print("sigma ok", flush=True)
if which in ("both", "pi"):
    plan.pi(t["dH"], t["G_less"], t["G_gtr"], o["P_less"], o["P_gtr"]); torch.cuda.synchronize(); print("pi ok", flush=True)
