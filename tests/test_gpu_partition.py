"""Partitioned (multi-GPU) path on ONE GPU: several rank views of a macro partition live in one
process; each computes its element contributions, packs the partial sums of the nodes it shares
(hhg_halo_pack), the test moves every send segment to the peer's receive segment (the transport
the library does with ncclSend/ncclRecv), and hhg_interface_sum_remote finishes the interface sum.
The assembled result must equal the unpartitioned epsilon_apply, and the owner-masked partial dots
must add up to the global dot.  Nothing here waits on another rank's kernels: every step is a
sequential kernel launch in one process.
"""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_2506_04157_b200 as hhg  # noqa: E402
from tests.harness import BC_SHELL, lib_eta, lib_mesh, lib_u, rel_l2  # noqa: E402
from workload import icoshell  # noqa: E402

C2 = (1e4, 10.0)


def _part_mesh(mac, level, tr, nparts, r):
    P = hhg.Mesh.part(mac, level, tr, nparts, r)
    P.blend_map(hhg.HHG_BLEND_SHELL)
    P.set_bc(hhg.HHG_BND_OUTER, hhg.HHG_BC_DIRICHLET0)
    P.set_bc(hhg.HHG_BND_INNER, hhg.HHG_BC_FREESLIP)
    return P


@pytest.mark.parametrize("nparts,level", [(2, 3), (4, 3), (8, 2)])
def test_partitioned_apply_matches_global(nparts, level):
    mac = icoshell(3, 2)
    M = lib_mesh(mac, level, True, BC_SHELL)
    eta = lib_eta(M, level, C2)
    u = lib_u(M, level, 2)
    y_ref = M.to_canonical(level, hhg.HHG_P2VEC, hhg.epsilon_apply(M, level, eta, u))
    eta_c = M.to_canonical(level, hhg.HHG_P1, eta)
    u_c = M.to_canonical(level, hhg.HHG_P2VEC, u)
    tr = hhg.partition_rcb(mac.verts, mac.tets, nparts)
    parts = [_part_mesh(mac, level, tr, nparts, r) for r in range(nparts)]
    ys, sends, infos = [], [], []
    for P in parts:
        e = P.from_canonical(level, hhg.HHG_P1, eta_c)
        uu = P.from_canonical(level, hhg.HHG_P2VEC, u_c)
        y = hhg.epsilon_apply_partial(P, level, e, uu)
        ys.append(y)
        sends.append(P.halo_pack(level, hhg.HHG_P2VEC, y))
        infos.append(P.halo_info(level, hhg.HHG_P2VEC))
    # transport: rank r's segment for neighbor q <- rank q's segment for neighbor r
    for r, P in enumerate(parts):
        nb, cnt = infos[r]
        off = np.concatenate([[0], np.cumsum(cnt)]) * 3
        recv = torch.zeros_like(sends[r])
        for i, q in enumerate(nb):
            nq, cq = infos[q]
            oq = np.concatenate([[0], np.cumsum(cq)]) * 3
            j = list(nq).index(r)
            recv[off[i]:off[i + 1]] = sends[q][oq[j]:oq[j + 1]]
        P.interface_sum_remote(level, hhg.HHG_P2VEC, recv, ys[r])
    covered = torch.zeros_like(y_ref)
    for r, P in enumerate(parts):
        yc = P.to_canonical(level, hhg.HHG_P2VEC, ys[r])
        mask = P.to_canonical(level, hhg.HHG_P2VEC, torch.ones_like(ys[r])) != 0
        assert rel_l2(yc[mask].cpu().numpy(), y_ref[mask].cpu().numpy()) <= 1e-14
        covered += mask.double()
    assert bool((covered > 0).all())
    # owner-masked dots over the parts add up to the global dot
    ref = float(hhg.hhg_dot(M, level, hhg.HHG_P2VEC, u, u).item())
    tot = 0.0
    for P in parts:
        uu = P.from_canonical(level, hhg.HHG_P2VEC, u_c)
        tot += float(hhg.hhg_dot(P, level, hhg.HHG_P2VEC, uu, uu).item())
    assert abs(tot - ref) <= 1e-13 * abs(ref)


def test_rank_without_macros_is_a_no_op():
    """Degenerate partition: every macro on rank 0, rank 1 empty.  The empty rank's vectors have length 0,
    its applies, interface sums and dots are no-ops (0 for the dot), it has no halo neighbours, and rank 0
    alone reproduces the global operator."""
    mac = icoshell(3, 2)
    level = 2
    tr = np.zeros(len(mac.tets), np.int32)
    E = _part_mesh(mac, level, tr, 2, 1)
    assert E.local_macros() == 0 and E.vec_len(level, hhg.HHG_P2VEC) == 0
    u = E.zeros(level, hhg.HHG_P2VEC)
    y = hhg.epsilon_apply_partial(E, level, E.zeros(level, hhg.HHG_P1), u)
    assert y.numel() == 0
    nb, cnt = E.halo_info(level, hhg.HHG_P2VEC)
    assert len(nb) == 0
    assert float(hhg.hhg_dot(E, level, hhg.HHG_P2VEC, u, u).item()) == 0.0
    F = _part_mesh(mac, level, tr, 2, 0)
    M = lib_mesh(mac, level, True, BC_SHELL)
    eta = lib_eta(M, level, C2)
    uu = lib_u(M, level, 2)
    ref = M.to_canonical(level, hhg.HHG_P2VEC, hhg.epsilon_apply(M, level, eta, uu))
    e = F.from_canonical(level, hhg.HHG_P1, M.to_canonical(level, hhg.HHG_P1, eta))
    v = F.from_canonical(level, hhg.HHG_P2VEC, M.to_canonical(level, hhg.HHG_P2VEC, uu))
    got = F.to_canonical(level, hhg.HHG_P2VEC, hhg.epsilon_apply(F, level, e, v))
    assert rel_l2(got.cpu().numpy(), ref.cpu().numpy()) <= 1e-14
