"""Quick timing probe: python tools/time_cfg.py cfg3 [reps]"""
import sys, time
sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import torch, qtgen, paper_1912_10024_b200 as qt
name = sys.argv[1] if len(sys.argv) > 1 else "small"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
p = qtgen.problem(name)
t0 = time.time()
t = qtgen.dev_inputs(p)
sh = p.shapes()
o = {k: torch.empty(sh["G" if k[0] == "S" else "D"], dtype=torch.complex128, device="cuda") for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
torch.cuda.synchronize(); print("gen", time.time() - t0, flush=True)
plan = qt.Plan(p); print(plan.info(), flush=True)
f = qt.count_flops(p)
for r in range(reps):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    e[0].record(); plan.sigma(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], o["S_less"], o["S_gtr"])
    e[1].record(); plan.pi(t["dH"], t["G_less"], t["G_gtr"], o["P_less"], o["P_gtr"]); e[2].record()
    torch.cuda.synchronize()
    ts, tp = e[0].elapsed_time(e[1]) / 1e3, e[1].elapsed_time(e[2]) / 1e3
    fs, fp = f["sigma_contraction"] + f["sigma_sandwich"], f["pi_contraction"] + f["pi_sandwich"]
    print(f"{name} rep{r}: sigma {ts:.3f}s {fs/ts/1e12:.2f} TF | pi {tp:.3f}s {fp/tp/1e12:.2f} TF | total {(fs+fp)/(ts+tp)/1e12:.2f} TF", flush=True)
