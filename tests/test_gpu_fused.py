"""GPU: the smoother / residual updates fused into the element kernel's write-out (launch_elem_epi)
(opt-in: HHG_EPI=1 at hierarchy creation; measured slower) against the default unfused path and the oracle.  Fused nodes (footprint interiors of
dense bricks) and consumer nodes (brick borders, macro interfaces, sparse bricks) together must reproduce the
unfused V-cycle to rounding (the same arithmetic per node; only the fp64 RED order on brick borders differs)."""
import os

import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_04157_b200 as hhg  # noqa: E402
from tests.harness import BC_SHELL, canon, lib_eta, lib_mesh, lib_u, oracle_case, rel_l2  # noqa: E402
from workload import icoshell, uniform_vec  # noqa: E402

C3 = (1e6, 30.0)


def _mg(M, levels, degree, no_epi):
    """no_epi=False: the fused epilogue (opt-in, HHG_EPI=1); True: the default unfused path."""
    etas = {L: lib_eta(M, L, C3) for L in levels}
    pv = {L: M.from_canonical(L, hhg.HHG_P2VEC, uniform_vec(M.canonical_keys(L, hhg.HHG_P2), 6)) for L in levels[1:]}
    if not no_epi:
        os.environ["HHG_EPI"] = "1"
    try:
        return hhg.MG(M, levels[0], levels[-1], etas, pv, pre=3, post=3, degree=degree, power_iters=20,
                      coarse_iters=50)
    finally:
        os.environ.pop("HHG_EPI", None)


@pytest.mark.parametrize("degree", [2, 3])
def test_fused_vcycle_equals_unfused_level4(degree):
    M = lib_mesh(icoshell(3, 2), 4, True, BC_SHELL)
    levels = (1, 2, 3, 4)
    mg, mg_ref = _mg(M, levels, degree, False), _mg(M, levels, degree, True)
    f = lib_u(M, 4, 4)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        x = mg.vcycle(f, stream=s)
        x_ref = mg_ref.vcycle(f, stream=s)
        xa, ita, rela = mg.ablock_cg(f, tol=1e-6, max_iters=100, stream=s)
        xb, itb, relb = mg_ref.ablock_cg(f, tol=1e-6, max_iters=100, stream=s)
    s.synchronize()
    e = float((x - x_ref).norm() / x_ref.norm())
    print(f"V(3,3) deg {degree} L4->1 fused vs unfused: {e:.2e}; A-block CG {ita} vs {itb} iterations")
    assert e <= 1e-13
    assert ita == itb and abs(rela - relb) <= 1e-6 * relb


def test_fused_vcycle_matches_oracle_level3():
    from oracle.multigrid import Hierarchy
    mac = icoshell(3, 2)
    discs, v0 = {}, {}
    for L in (1, 2, 3):
        lm, d, _ = oracle_case(mac, L, True, BC_SHELL, C3, 0.0, build=("A",))
        discs[L], v0[L] = d, uniform_vec(lm.p2_keys, 6)
    H = Hierarchy(discs, v0, pre=3, post=3, degree=3, power_iters=20, coarse_iters=50)
    x_o = H.vcycle(discs[3].project(uniform_vec(discs[3].lm.p2_keys, 4)))
    M = lib_mesh(mac, 3, True, BC_SHELL)
    mg = _mg(M, (1, 2, 3), 3, False)
    x = mg.vcycle(lib_u(M, 3, 4))
    torch.cuda.synchronize()
    e = rel_l2(canon(M, 3, hhg.HHG_P2VEC, x), x_o)
    print(f"fused V-cycle L3->1 vs oracle {e:.2e}")
    assert e <= 1e-9
