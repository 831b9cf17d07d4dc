"""Out-of-bounds and contract guards of our own (compute-sanitizer is closed on this GPU pool):
every tensor the library touches is a view into a larger allocation whose margins hold a canary pattern; after
the call the margins must be unchanged (no write outside a tensor), the inputs must be bit-identical to their
copies (inputs are never modified: qt_sse.h), and every output element must have been written (outputs start
as NaN). Covers FP64 / FP32, separate / fused calls, many-chunk workspaces, the deterministic flag, a loopback
rank of a 2-D grid, shift_step > 1, and the RGF solver."""
from __future__ import annotations

import numpy as np
import pytest

import qtgen
from qtgen import rgf as grgf
from tests.helpers import micro

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1912_10024_b200 as qt  # noqa: E402

MARGIN = 4096   # complex elements on each side (64 KB)
CANARY = complex(1.2345678e300, -9.87654321e-300)


class Guarded:
    def __init__(self):
        self.bufs = []

    def make(self, shape, fill=None):
        n = int(np.prod(shape))
        buf = torch.full((n + 2 * MARGIN,), CANARY, dtype=torch.complex128, device="cuda")
        view = buf[MARGIN:MARGIN + n].view(shape)
        if fill is not None:
            view.copy_(fill)
        else:
            view.fill_(complex(float("nan"), float("nan")))
        self.bufs.append(buf)
        return view

    def check_margins(self):
        for buf in self.bufs:
            m = torch.cat([buf[:MARGIN], buf[-MARGIN:]])
            assert bool((m == CANARY).all()), "write outside a tensor's bounds"


def _inputs(p, g, t):
    return {k: g.make(v.shape, v) for k, v in t.items()}


@pytest.mark.parametrize("prec", [qt.QT_PREC_FP64, qt.QT_PREC_FP32_MIXED])
@pytest.mark.parametrize("fused,ws,flags", [(False, 0, 0), (True, 1, 0), (True, 1, qt.QT_FLAG_DETERMINISTIC)])
def test_guarded_single(prec, fused, ws, flags):
    for p in (qtgen.problem("tiny"), micro(Na=6, Nb=3, Norb=3, NE=20, Nw=4, Nkz=3, fill=0.8, seed=3)):
        if p.name == "micro":
            p.shift_step = 2
        t = qtgen.dev_inputs(p)
        g = Guarded()
        ins = _inputs(p, g, t)
        sh = p.shapes()
        out = {k: g.make(sh["G" if k[0] == "S" else "D"]) for k in ("S_less", "S_gtr", "P_less", "P_gtr")}
        plan = qt.Plan(p, precision=prec, workspace_limit=ws, flags=flags)
        if fused:
            plan.sigma_pi(ins["dH"], ins["G_less"], ins["G_gtr"], ins["D_less"], ins["D_gtr"], out["S_less"],
                          out["S_gtr"], out["P_less"], out["P_gtr"])
        else:
            plan.sigma(ins["dH"], ins["G_less"], ins["G_gtr"], ins["D_less"], ins["D_gtr"], out["S_less"], out["S_gtr"])
            plan.pi(ins["dH"], ins["G_less"], ins["G_gtr"], out["P_less"], out["P_gtr"])
        torch.cuda.synchronize()
        plan.close()
        g.check_margins()
        for k in ins:
            assert torch.equal(ins[k], t[k]), f"input {k} modified"
        for k in out:
            assert not torch.isnan(out[k]).any(), f"{k}: elements never written"


def test_guarded_loopback_rank():
    p = qtgen.problem("tiny")
    t = qtgen.dev_inputs(p)
    for r in range(4):
        plan = qt.Plan(p, rank=r, nranks=4, shard=qt.QT_SHARD_2D, grid_atoms=2)
        i = plan.info()
        w, ew = slice(i["w_lo"], i["w_hi"]), slice(i["ew_lo"], i["ew_hi"])
        g = Guarded()
        win = {k: g.make(t[k][:, ew, w].shape, t[k][:, ew, w]) for k in ("G_less", "G_gtr")}
        win.update({k: g.make(t[k][:, :, w].shape, t[k][:, :, w]) for k in ("D_less", "D_gtr")})
        dH = g.make(t["dH"][w].shape, t["dH"][w])
        nout, neo = i["a_hi"] - i["a_lo"], i["e_hi"] - i["e_lo"]
        S = [g.make((p.Nkz, neo, nout, p.Norb, p.Norb)) for _ in range(2)]
        P = [g.make((p.Nqz, p.Nw, nout, p.Nb + 1, 3, 3)) for _ in range(2)]
        plan.sigma_pi(dH, win["G_less"], win["G_gtr"], win["D_less"], win["D_gtr"], S[0], S[1], P[0], P[1])
        torch.cuda.synchronize()
        plan.close()
        g.check_margins()
        for x in S + P:
            assert not torch.isnan(x).any()


def test_guarded_rgf():
    r = grgf.RgfProblem(P=3, bnum=4, bs=20)
    t = {k: torch.from_numpy(v).cuda() for k, v in grgf.host_inputs(r).items()}
    g = Guarded()
    ins = {k: g.make(v.shape, v) for k, v in t.items()}
    out = {k: g.make(t["Ad"].shape) for k in ("GR", "GL", "GG")}
    plan = qt.Rgf(r.P, r.bnum, r.bs)
    plan.solve(ins["Ad"], ins["Au"], ins["Al"], ins["Sl"], ins["Sg"], out["GR"], out["GL"], out["GG"])
    assert plan.check() is None
    plan.close()
    g.check_margins()
    for k in ins:
        assert torch.equal(ins[k], t[k])
    for k in out:
        assert not torch.isnan(out[k]).any()
