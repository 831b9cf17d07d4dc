"""FP32 mixed mode vs the oracle on small problems: python tools/debug_fp32.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, qtgen, oracle
import paper_1912_10024_b200 as qt
from tests.helpers import MICROS, micro, inputs, rel_fro

def check(p, seed=1):
    inp = inputs(p, seed=seed)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    out = qt.run(p, t, 1j, -1j, precision=qt.QT_PREC_FP32_MIXED)
    torch.cuda.synchronize()
    SL, SG = oracle.sigma(p, inp, 1j)
    PL, PG = oracle.pi(p, inp, -1j)
    e = [rel_fro(out["S_less"].cpu().numpy(), SL, (-2, -1)), rel_fro(out["S_gtr"].cpu().numpy(), SG, (-2, -1)),
         rel_fro(out["P_less"].cpu().numpy(), PL, (-2, -1)), rel_fro(out["P_gtr"].cpu().numpy(), PG, (-2, -1))]
    print(p.Na, p.Nb, p.Norb, p.NE, p.Nw, p.Nkz, "errors S<,S>,P<,P>:", ["%.2e" % x for x in e], flush=True)

if len(sys.argv) == 1:
  check(qtgen.problem("tiny"))
  for i, m in enumerate(MICROS):
    if m.get("Norb", 3) <= 10:
        check(micro(**m), seed=10 + i)
  check(micro(Na=7, Nb=4, Norb=10, NE=13, Nw=3, Nkz=3, fill=0.7, seed=10))
if len(sys.argv) > 1 and sys.argv[1] == "norb":
    for Norb in range(1, 11):
        check(micro(Na=7, Nb=4, Norb=Norb, NE=13, Nw=3, Nkz=3, fill=0.7, seed=Norb), seed=Norb)
