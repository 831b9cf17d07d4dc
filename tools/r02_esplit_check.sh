#!/bin/bash
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_loopback.py tests/test_gpu_guard.py tests/test_gpu_fp32.py -m "gpu and not slow" -x -q > gpurun_out/r02_pytest_esplit.log 2>&1
echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_esplit.log
python tools/kt.py prof
python - <<'PY'
import sys; sys.path.insert(0, '.')
import torch, qtgen, paper_1912_10024_b200 as qt
p = qtgen.problem("prof4")
t = qtgen.dev_inputs(p); sh = p.shapes()
o = {k: torch.empty(sh["G" if k[0] == "S" else "D"], dtype=torch.complex128, device="cuda") for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
f = qt.count_flops(p)["total"]
for ws in (1 << 30, 0):
    plan = qt.Plan(p, workspace_limit=ws)
    plan.sigma_pi(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], o["S_less"], o["S_gtr"], o["P_less"], o["P_gtr"])
    torch.cuda.synchronize()
    plan.timing(True); plan.timing_read()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); plan.sigma_pi(t["dH"], t["G_less"], t["G_gtr"], t["D_less"], t["D_gtr"], o["S_less"], o["S_gtr"], o["P_less"], o["P_gtr"]); e1.record()
    torch.cuda.synchronize(); ms = e0.elapsed_time(e1)
    r = plan.timing_read()
    print("prof4 ws", ws >> 30, "GB:", round(ms, 1), "ms", round(f / ms / 1e9, 2), "TF", {k: (round(v[0], 1), v[1]) for k, v in r.items() if v[1]})
    plan.close()
PY
