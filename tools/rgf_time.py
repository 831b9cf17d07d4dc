"""RGF timing probe: python tools/rgf_time.py rgf_finfet [reps]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1912_10024_b200 as qt
from qtgen import rgf as grgf
p = grgf.problem(sys.argv[1] if len(sys.argv) > 1 else "rgf_finfet")
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time(); t = grgf.dev_inputs(p); torch.cuda.synchronize(); print("gen", round(time.time() - t0, 1), "s", flush=True)
plan = qt.Rgf(p.P, p.bnum, p.bs)
out = {k: torch.empty_like(t["Ad"]) for k in ("GR", "GL", "GG")}
f = qt.rgf_count_flops(p.P, p.bnum, p.bs)
for r in range(reps):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.solve(t["Ad"], t["Au"], t["Al"], t["Sl"], t["Sg"], out["GR"], out["GL"], out["GG"]); e1.record()
    torch.cuda.synchronize(); ms = e0.elapsed_time(e1)
    print(f"{p.name} rep{r}: {ms:.1f} ms  executed {f['executed'] / ms / 1e9:.2f} TF  paper-model {f['paper_model'] / ms / 1e9:.2f} TF",
          "singular:", plan.check(), flush=True)
