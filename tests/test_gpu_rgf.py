"""GPU parity of the RGF solver (include/qt_rgf.h) against the dense CPU oracle of Eq. 1
(oracle/rgf.py), through the C ABI. Bar: per diagonal block, relative Frobenius error ≤ 1e-10 (SPEC S:249 uses
1e-10 for RGF ≡ dense inverse; the inversions amplify rounding by the blocks' condition numbers, so FP64 RGF is
not held to the SSE's 1e-12). At the bench size, where the dense oracle (N = 48,640) is out of reach, the
properties that hold at any size are checked on every block: G^> − G^< = G^R − G^A (η = 0) and
anti-Hermiticity of G^≷."""
from __future__ import annotations

import numpy as np
import pytest

from oracle import rgf as orgf
from qtgen import rgf as grgf
from tests.helpers import rel_fro

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import paper_1912_10024_b200 as qt  # noqa: E402

TOL = 1e-10
AX = (-2, -1)


def _run(inp):
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    out = qt.rgf_run(t)
    torch.cuda.synchronize()
    return {k: v.cpu().numpy() for k, v in out.items()}


@pytest.mark.parametrize("name", ["rgf_tiny", "rgf_small", "rgf_mid"])
def test_rgf_matches_dense_oracle(name):
    p = grgf.problem(name)
    inp = grgf.host_inputs(p, seed=11)
    g = _run(inp)
    GR, GL, GG = orgf.solve(inp)
    for got, ref in ((g["GR"], GR), (g["GL"], GL), (g["GG"], GG)):
        assert rel_fro(got, ref, AX) <= TOL


@pytest.mark.parametrize("bnum,bs", [(1, 16), (2, 5), (3, 33), (5, 1)])
def test_rgf_shapes(bnum, bs):
    """bnum = 1 (no recursion), odd block sizes, scalar blocks."""
    p = grgf.RgfProblem(P=3, bnum=bnum, bs=bs)
    inp = grgf.host_inputs(p, seed=bnum * 100 + bs)
    g = _run(inp)
    GR, GL, GG = orgf.solve(inp)
    for got, ref in ((g["GR"], GR), (g["GL"], GL), (g["GG"], GG)):
        assert rel_fro(got, ref, AX) <= TOL


def test_rgf_singular_block_reported():
    p = grgf.RgfProblem(P=2, bnum=3, bs=4)
    inp = grgf.host_inputs(p, seed=1)
    inp["Ad"][1, 0] = 0.0            # point 1, block 0: singular pivot
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda() for k, v in inp.items()}
    with pytest.raises(qt.QTError, match="singular pivot block 0 at point 1"):
        qt.rgf_run(t)


@pytest.mark.slow
def test_rgf_bench_size_properties():
    """rgf_finfet (76 blocks of 640, 16 points) with η = 0: G^> − G^< = G^R − G^A and anti-Hermitian G^≷ on
    every block (device-side checks)."""
    p = grgf.problem("rgf_finfet")
    t = grgf.dev_inputs(p, eta=0.0)
    out = qt.rgf_run(t)
    del t
    GA = out["GR"].transpose(-1, -2).conj()
    lhs = (out["GG"] - out["GL"]) - (out["GR"] - GA)
    scale = out["GR"].abs().amax(dim=(-2, -1))
    assert float((lhs.abs().amax(dim=(-2, -1)) / scale).max()) < 1e-10
    for G in (out["GL"], out["GG"]):
        ah = (G + G.transpose(-1, -2).conj()).abs().amax(dim=(-2, -1)) / G.abs().amax(dim=(-2, -1))
        assert float(ah.max()) < 1e-10
