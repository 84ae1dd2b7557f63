"""Multi-GPU host logic: macro partition, owner masks, cross-rank interface plans.

These run on CPU (no GPU needed: partitioning and plan building are host-only library calls).
The world-size-2 test runs two gloo processes that each build their own rank's plan and exchange
per-slot values in the order the plan prescribes -- the same protocol the library drives with
ncclSend/ncclRecv -- and check that every slot received the peer's value for the same node.
"""
import os

import numpy as np
import pytest

import paper_2506_04157_b200 as hhg
from workload import icoshell, reference_tet
from workload.seeded import hash_keys


def _parts(mac, level_max, nparts):
    tr = hhg.partition_rcb(mac.verts, mac.tets, nparts, radial=True)
    return tr, [hhg.Mesh.part(mac, level_max, tr, nparts, r) for r in range(nparts)]


@pytest.mark.parametrize("nparts", [2, 4, 8])
def test_rcb_partition_is_balanced(nparts):
    mac = icoshell(3, 2)
    tr = hhg.partition_rcb(mac.verts, mac.tets, nparts)
    counts = np.bincount(tr, minlength=nparts)
    assert counts.sum() == len(mac.tets) and counts.min() == counts.max() == len(mac.tets) // nparts
    # deterministic
    assert np.array_equal(tr, hhg.partition_rcb(mac.verts, mac.tets, nparts))


@pytest.mark.parametrize("nparts,level", [(2, 2), (4, 1), (8, 2)])
@pytest.mark.parametrize("space", [hhg.HHG_P1, hhg.HHG_P2])
def test_owner_masks_count_every_node_once(nparts, level, space):
    mac = icoshell(3, 2)
    tr, parts = _parts(mac, level, nparts)
    total = sum(p.owned_count(level, space) for p in parts)
    assert total == parts[0].canonical_len(level, space)
    for r, p in enumerate(parts):
        assert p.rank() == (r, nparts)
        assert p.local_macros() == int((tr == r).sum())


@pytest.mark.parametrize("nparts,level", [(2, 2), (4, 2), (8, 1)])
def test_halo_plans_are_symmetric(nparts, level):
    """Rank r lists q as neighbor iff q lists r, with the same shared nodes in the same order, and a
    node is shared with q iff q's macros contain it."""
    mac = icoshell(3, 2)
    tr, parts = _parts(mac, level, nparts)
    for space in (hhg.HHG_P1, hhg.HHG_P2VEC):
        info = [p.halo_info(level, space) for p in parts]
        keys = [p.halo_keys(level, space) for p in parts]
        for r in range(nparts):
            nb, cnt = info[r]
            off = np.concatenate([[0], np.cumsum(cnt)])
            for i, q in enumerate(nb):
                assert q != r
                nq, cq = info[q]
                j = list(nq).index(r)
                offq = np.concatenate([[0], np.cumsum(cq)])
                assert cq[j] == cnt[i]
                assert np.array_equal(keys[r][off[i]:off[i + 1]], keys[q][offq[j]:offq[j + 1]])
        # every shared node is a macro-boundary node (dim <= 2) and appears once per neighbor
        for r in range(nparts):
            nb, cnt = info[r]
            off = np.concatenate([[0], np.cumsum(cnt)])
            assert (keys[r][:, 0] <= 2).all()
            for i in range(len(nb)):
                seg = keys[r][off[i]:off[i + 1]]
                assert len({tuple(k) for k in seg}) == len(seg)


def test_single_rank_has_no_halo():
    M = hhg.Mesh.from_macro(reference_tet(), 2)
    nb, cnt = M.halo_info(2, hhg.HHG_P2VEC)
    assert len(nb) == 0 and M.owned_count(2, hhg.HHG_P2) == M.canonical_len(2, hhg.HHG_P2)


def test_part_without_comm_needs_tet_rank_and_valid_ranks():
    mac = icoshell(3, 2)
    tr = hhg.partition_rcb(mac.verts, mac.tets, 2)
    with pytest.raises(hhg.HHGError):
        hhg.Mesh(mac.verts, mac.tets, mac.vtag, 1, tet_rank=tr)        # partition without comm
    with pytest.raises(hhg.HHGError):
        hhg.Mesh.part(mac, 1, tr, 2, 2)                                # rank out of range
    with pytest.raises(hhg.HHGError):
        hhg.Mesh.part(mac, 1, np.full(len(mac.tets), 3, np.int32), 2, 0)


# ------------------------------------------------------------------ world size 2 over gloo
def _exchange_worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        mac = icoshell(3, 2)
        level = 2
        tr = hhg.partition_rcb(mac.verts, mac.tets, world)
        M = hhg.Mesh.part(mac, level, tr, world, rank)
        ok = True
        for space, nc in ((hhg.HHG_P1, 1), (hhg.HHG_P2VEC, 3)):
            nb, cnt = M.halo_info(level, space)
            keys = M.halo_keys(level, space)
            off = np.concatenate([[0], np.cumsum(cnt)])
            # what each rank "sends" for a node: a value only the node key and the sender determine
            send = np.stack([hash_keys(keys, 100 + rank, c) for c in range(nc)], 1).astype(np.float64)
            recv = np.zeros_like(send)
            reqs = []
            for i, q in enumerate(nb):
                s = torch.from_numpy(np.ascontiguousarray(send[off[i]:off[i + 1]]))
                rbuf = torch.zeros_like(s)
                reqs.append((dist.isend(s, int(q)), dist.irecv(rbuf, int(q)), i, rbuf))
            for a, b, i, rbuf in reqs:
                a.wait()
                b.wait()
                recv[off[i]:off[i + 1]] = rbuf.numpy()
            for i, q in enumerate(nb):
                expect = np.stack([hash_keys(keys[off[i]:off[i + 1]], 100 + int(q), c) for c in range(nc)], 1)
                ok &= bool(np.array_equal(recv[off[i]:off[i + 1]], expect))
            ok &= len(nb) == world - 1
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


def test_world2_gloo_exchange_protocol():
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0, 0])
    procs = [ctx.Process(target=_exchange_worker, args=(r, 2, port, out)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(120)
    assert all(p.exitcode == 0 for p in procs)
    assert list(out) == [1, 1]


# ------------------------------------------------------------------ the library's host-staged transport callbacks
def _hostcomm_worker(rank, world, port, out):
    """The HostComm trampolines the library calls (hhg_comm_create_host), driven with the halo plans the
    library built for this rank: every neighbour's block arrives in the right slots, allreduce sums."""
    import ctypes
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        comm = hhg.HostComm()
        exchange, allreduce = comm._cb
        mac = icoshell(3, 2)
        level = 2
        tr = hhg.partition_rcb(mac.verts, mac.tets, world)
        M = hhg.Mesh.part(mac, level, tr, world, rank)
        ok = True
        for space, nc in ((hhg.HHG_P1, 1), (hhg.HHG_P2VEC, 3)):
            nb, cnt = M.halo_info(level, space)
            keys = M.halo_keys(level, space)
            off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.int64)
            send = np.ascontiguousarray(np.stack([hash_keys(keys, 100 + rank, c) for c in range(nc)], 1).astype(np.float64))
            recv = np.zeros_like(send)
            nbr = np.ascontiguousarray(nb, dtype=np.int32)
            rc = exchange(None, len(nbr), nbr.ctypes.data_as(ctypes.POINTER(ctypes.c_int)),
                          off.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)), nc,
                          send.ctypes.data_as(ctypes.POINTER(ctypes.c_double)),
                          recv.ctypes.data_as(ctypes.POINTER(ctypes.c_double)))
            ok &= rc == 0
            for i, q in enumerate(nb):
                expect = np.stack([hash_keys(keys[off[i]:off[i + 1]], 100 + int(q), c) for c in range(nc)], 1)
                ok &= bool(np.array_equal(recv[off[i]:off[i + 1]], expect))
        v = np.array([rank + 1.0, 10.0 * rank], dtype=np.float64)
        ok &= allreduce(None, v.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), 2) == 0
        ok &= bool(np.array_equal(v, [world * (world + 1) / 2.0, 10.0 * world * (world - 1) / 2.0]))
        out[rank] = 1 if ok else 0
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_host_transport_callbacks_gloo(world):
    import socket
    import torch.multiprocessing as mp
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    ctx = mp.get_context("spawn")
    out = ctx.Array("i", [0] * world)
    procs = [ctx.Process(target=_hostcomm_worker, args=(r, world, port, out)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(180)
    assert all(p.exitcode == 0 for p in procs)
    assert list(out) == [1] * world
