"""per-kernel times for one sigma+pi call pair: python tools/kt.py prof [fp32]"""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, qtgen, paper_1912_10024_b200 as qt
p = qtgen.problem(sys.argv[1] if len(sys.argv) > 1 else "prof"); t = qtgen.dev_inputs(p); sh = p.shapes()
prec = qt.QT_PREC_FP32_MIXED if "fp32" in sys.argv[2:] else qt.QT_PREC_FP64
o = {k: torch.empty(sh["G" if k[0] == "S" else "D"], dtype=torch.complex128, device="cuda") for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
plan = qt.Plan(p, precision=prec)
def run():
    plan.sigma(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], o["S_less"], o["S_gtr"])
    plan.pi(t["dH"], t["G_less"], t["G_gtr"], o["P_less"], o["P_gtr"])
run(); torch.cuda.synchronize()
plan.timing(True); plan.timing_read(); run()
r = plan.timing_read(); f = qt.count_flops(p)
tot = sum(v[0] for v in r.values())
print({k: round(v[0], 1) for k, v in r.items() if v[1]}, "total ms", round(tot, 1), "TF", round(f["total"] / tot / 1e9, 2))
