"""Thin ctypes binding of libhhgstokes.so (include/hhg_stokes.h) -- argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; PyTorch supplies device
memory (tensors), the current CUDA stream and process groups.  There is NO CPU fallback:
importing this package raises if the shared library is missing, and every call raises
``HHGError`` with the library's message on failure.

Names follow the C-ABI (and the paper's notation): ``hhg_mesh_create`` -> ``Mesh``,
``blend_map``, ``epsilon_apply``, ``div_apply``, ``divT_apply``, ``stokes_apply``,
``hhg_diag``, ``hhg_dot``, ``p2_restrict``, ``p2_prolong``, ``chebyshev_smooth``,
``hhg_power_iteration``, ``MG`` (``hhg_mg_create``) with ``vcycle``.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HHG_LIB") or os.path.join(_HERE, "lib", "libhhgstokes.so")  # HHG_LIB: A/B builds

HHG_P1, HHG_P2, HHG_P2VEC = 1, 2, 3
HHG_BLEND_IDENTITY, HHG_BLEND_SHELL = 0, 1
HHG_BND_ALL, HHG_BND_INNER, HHG_BND_OUTER = 0, 1, 2
HHG_BC_NONE, HHG_BC_DIRICHLET0, HHG_BC_FREESLIP = 0, 1, 2
HHG_VISC_FULL, HHG_VISC_EPS = 0, 1

ERRORS = {-1: "HHG_EINVAL", -2: "HHG_ELEVEL", -3: "HHG_ENOTREADY", -4: "HHG_EZEROOP", -5: "HHG_EDOMAIN",
          -6: "HHG_ECUDA", -7: "HHG_ENCCL", -8: "HHG_ENOMEM"}

# every symbol declared in include/hhg_stokes.h
EXPORTS = [
    "hhg_last_error", "hhg_version", "hhg_comm_unique_id", "hhg_comm_create", "hhg_comm_destroy",
    "hhg_mesh_create", "hhg_mesh_destroy", "hhg_mesh_local_macros", "blend_map", "hhg_set_bc",
    "hhg_vec_len", "hhg_canonical_len", "hhg_canonical_keys", "hhg_to_canonical", "hhg_from_canonical",
    "hhg_node_coords", "hhg_apply_bc", "hhg_interface_sum", "epsilon_apply", "div_apply", "divT_apply",
    "stokes_apply", "hhg_diag", "hhg_dot", "p2_restrict", "p2_prolong", "chebyshev_smooth",
    "hhg_power_iteration", "hhg_mg_create", "hhg_mg_lambda", "hhg_mg_coarse_iterations", "vcycle", "vcycle_host", "hhg_mg_profile",
    "hhg_mg_profile_get", "hhg_mg_profile_get_dense", "hhg_mg_destroy", "hhg_launch_count",
    "hhg_mesh_create_part", "hhg_partition_rcb", "hhg_mesh_rank", "hhg_halo_info", "hhg_halo_keys",
    "hhg_owned_count", "hhg_halo_pack", "hhg_interface_sum_remote", "epsilon_apply_partial",
    "hhg_ablock_cg", "hhg_mass_apply", "hhg_mass_diag", "hhg_stokes_create", "hhg_stokes_solve",
    "hhg_stokes_destroy", "hhg_buoyancy_load", "hhg_icoshell_macro", "hhg_mesh_create_icoshell",
    "hhg_mg_create_qeta", "epsilon_apply_qeta", "hhg_diag_qeta",
    "hhg_stokes_schur_apply", "hhg_kp1_apply", "hhg_kp1_diag", "hhg_vmass_apply", "hhg_vmass_diag",
    "p1_prolong", "p1_restrict", "hhg_kmg_create", "hhg_kmg_solve", "hhg_kmg_destroy",
    "hhg_temp_apply", "hhg_temp_solver_create", "hhg_temp_solve", "hhg_temp_solver_destroy", "hhg_mmoc",
    "vcycle_host_batch", "hhg_set_deterministic", "hhg_mesh_prepare", "hhg_comm_create_host",
]


class HHGError(RuntimeError):
    pass


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"libhhgstokes.so not built ({LIB_PATH}); run `python __graft_entry__.py build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    P, I, I64, D = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64, ctypes.c_double
    sig = {
        "hhg_last_error": ([], ctypes.c_char_p), "hhg_version": ([], ctypes.c_char_p),
        "hhg_launch_count": ([I], I64),
        "hhg_comm_unique_id": ([P], I), "hhg_comm_create": ([P, I, I, I, P], I), "hhg_comm_destroy": ([P], I),
        "hhg_mesh_create": ([P, I64, P, I64, P, I, P, P, P], I), "hhg_mesh_destroy": ([P], I),
        "hhg_mesh_local_macros": ([P, P], I), "blend_map": ([P, I], I), "hhg_set_bc": ([P, I, I], I),
        "hhg_vec_len": ([P, I, I, P], I), "hhg_canonical_len": ([P, I, I, P], I),
        "hhg_canonical_keys": ([P, I, I, P], I), "hhg_to_canonical": ([P, I, I, P, P, P], I),
        "hhg_from_canonical": ([P, I, I, P, P, P], I), "hhg_node_coords": ([P, I, I, P, P], I),
        "hhg_apply_bc": ([P, I, P, P], I), "hhg_interface_sum": ([P, I, I, P, P], I),
        "epsilon_apply": ([P, I, I, P, P, P, P], I), "div_apply": ([P, I, D, P, P, P], I),
        "divT_apply": ([P, I, P, P, I, P], I), "stokes_apply": ([P, I, P, D, P, P, P, P, P], I),
        "hhg_diag": ([P, I, P, P, P], I), "hhg_dot": ([P, I, I, P, P, P, P], I),
        "p2_restrict": ([P, I, P, P, P], I), "p2_prolong": ([P, I, P, P, P], I),
        "chebyshev_smooth": ([P, I, P, P, I, D, D, P, P, P, P], I),
        "hhg_power_iteration": ([P, I, P, P, I, P, P, P], I),
        "hhg_mg_create": ([P, P, P, P, P], I), "hhg_mg_lambda": ([P, I, P], I), "hhg_mg_coarse_iterations": ([P, P], I), "vcycle": ([P, P, P, P], I),
        "vcycle_host": ([P, P, P, P], I), "hhg_mg_profile": ([P, I], I),
        "hhg_mg_profile_get": ([P, P, P, P, P], I), "hhg_mg_profile_get_dense": ([P, P], I),
        "hhg_mg_destroy": ([P], I),
        "hhg_mesh_create_part": ([P, I64, P, I64, P, I, P, I, I, P], I),
        "hhg_partition_rcb": ([P, I64, P, I64, I, I, P], I), "hhg_mesh_rank": ([P, P, P], I),
        "hhg_halo_info": ([P, I, I, P, P, P], I), "hhg_halo_keys": ([P, I, I, P], I),
        "hhg_owned_count": ([P, I, I, P], I), "hhg_halo_pack": ([P, I, I, P, P, P], I),
        "hhg_interface_sum_remote": ([P, I, I, P, P, P], I), "epsilon_apply_partial": ([P, I, I, P, P, P, P], I),
        "hhg_ablock_cg": ([P, P, P, D, I, P, P, P], I),
        "hhg_mass_apply": ([P, I, P, P, P, P], I), "hhg_mass_diag": ([P, I, P, P, P], I),
        "hhg_stokes_create": ([P, P, P, D, P, P], I), "hhg_stokes_solve": ([P, P, P, P, P, P], I),
        "hhg_stokes_destroy": ([P], I), "hhg_buoyancy_load": ([P, I, P, P, P], I),
        "hhg_icoshell_macro": ([I, I, D, D, P, P, P, P, P], I),
        "hhg_mesh_create_icoshell": ([I, I, D, D, I, P, P, P], I),
        "hhg_mg_create_qeta": ([P, P, P, P, P, P], I), "epsilon_apply_qeta": ([P, I, P, D, D, D, P, P, P], I),
        "hhg_diag_qeta": ([P, I, P, D, D, D, P, P], I),
        "hhg_stokes_schur_apply": ([P, P, P, P], I),
        "hhg_kp1_apply": ([P, I, P, D, P, P, P], I), "hhg_kp1_diag": ([P, I, P, D, P, P], I),
        "hhg_vmass_apply": ([P, I, P, D, P, P, P], I), "hhg_vmass_diag": ([P, I, P, D, P, P], I),
        "p1_prolong": ([P, I, P, P, P], I), "p1_restrict": ([P, I, P, P, P], I),
        "hhg_kmg_create": ([P, P, P, D, P], I), "hhg_kmg_solve": ([P, P, P, D, D, I, P, P, P], I),
        "hhg_kmg_destroy": ([P], I),
        "hhg_temp_apply": ([P, I, P, P, P, P, I, P], I), "hhg_temp_solver_create": ([P, I, P, I, P], I),
        "hhg_temp_solve": ([P, P, P, P, D, D, I, D, I, P, P, P], I), "hhg_temp_solver_destroy": ([P], I),
        "hhg_mmoc": ([P, I, P, P, P, D, P, P], I),
        "vcycle_host_batch": ([P, P, P, I, P], I),
        "hhg_set_deterministic": ([P, I], I), "hhg_mesh_prepare": ([P], I),
        "hhg_comm_create_host": ([I, I, P, P, P, P], I),
    }
    for name, (args, res) in sig.items():
        f = getattr(lib, name)
        f.argtypes = args
        f.restype = res
    return lib


_lib = _load()


def lib():
    return _lib


def _chk(rc):
    if rc != 0:
        raise HHGError(f"{ERRORS.get(rc, rc)}: {_lib.hhg_last_error().decode()}")


def _ptr(t):
    if t is None:
        return None
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    return t.data_ptr()


def _dev(t, n=None, name="tensor"):
    import torch
    if t is None:
        return None
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise HHGError(f"{name}: need a contiguous float64 CUDA tensor")
    if n is not None and t.numel() != n:
        raise HHGError(f"{name}: length {t.numel()} != expected {n}")
    if t.numel() == 0:       # empty vector (a rank without macros): any valid device address, never read
        return _empty_device_ptr()
    return t.data_ptr()


_EMPTY = []


def _empty_device_ptr():
    import torch
    if not _EMPTY:
        _EMPTY.append(torch.zeros(1, dtype=torch.float64, device="cuda"))
    return _EMPTY[0].data_ptr()


def _stream(stream=None):
    """The CUDA stream a call runs on (default: torch's current stream).  When it is not the default
    stream, it first waits for the default stream, where tensors made outside a `torch.cuda.stream`
    block are produced (torch's side streams are non-blocking: without the wait a call could read an
    input that is still being written)."""
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    d = torch.cuda.default_stream(s.device)
    if s != d:
        s.wait_stream(d)
    return ctypes.c_void_p(s.cuda_stream)


def version() -> str:
    return _lib.hhg_version().decode()


def launch_count(reset=False) -> int:
    return int(_lib.hhg_launch_count(1 if reset else 0))


class Comm:
    """hhg_comm_create: the library's own NCCL communicator (one process per GPU); the unique id is
    made on rank 0 and broadcast through the caller's torch.distributed process group."""

    def __init__(self, rank, world, device=0, group=None):
        import torch
        import torch.distributed as dist
        idb = np.zeros(128, dtype=np.uint8)
        if rank == 0:
            _chk(_lib.hhg_comm_unique_id(_ptr(idb)))
        t = torch.from_numpy(idb.astype(np.int64))
        if dist.get_backend(group) == "nccl":
            t = t.cuda()
        dist.broadcast(t, 0, group=group)
        idb = t.cpu().numpy().astype(np.uint8)
        h = ctypes.c_void_p()
        _chk(_lib.hhg_comm_create(_ptr(idb), int(world), int(rank), int(device), ctypes.byref(h)))
        self.handle, self.rank, self.world = h, rank, world

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_comm_destroy(self.handle)
            self.handle = None


_EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(ctypes.c_int),
                                ctypes.POINTER(ctypes.c_int64), ctypes.c_int, ctypes.POINTER(ctypes.c_double),
                                ctypes.POINTER(ctypes.c_double))
_ALLREDUCE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.POINTER(ctypes.c_double), ctypes.c_int64)


class HostComm:
    """hhg_comm_create_host: the library's interface exchange and allreduce carried by a torch.distributed
    process group (e.g. gloo) through host memory -- any number of ranks may share one GPU.  The callbacks
    only move bytes (isend/irecv of the library's packed partial sums, all_reduce of its scalars)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.group = group
        self.rank, self.world = dist.get_rank(group), dist.get_world_size(group)

        def exchange(user, n_nbr, nbr, off, nc, send, recv):
            try:
                n = int(off[n_nbr]) * nc if n_nbr > 0 else 0
                if n == 0:
                    return 0
                sv = torch.from_numpy(np.ctypeslib.as_array(send, shape=(n,)))
                rv = torch.from_numpy(np.ctypeslib.as_array(recv, shape=(n,)))
                reqs = []
                for i in range(n_nbr):
                    a, b = int(off[i]) * nc, int(off[i + 1]) * nc
                    peer = dist.get_global_rank(group, int(nbr[i])) if group is not None else int(nbr[i])
                    reqs.append(dist.isend(sv[a:b].clone(), peer, group=group))
                    reqs.append(dist.irecv(rv[a:b], peer, group=group))
                for r in reqs:
                    r.wait()
                return 0
            except Exception as e:  # pragma: no cover - reported through HHG_ENCCL
                print("HostComm exchange failed:", e)
                return 1

        def allreduce(user, buf, n):
            try:
                if n > 0:
                    dist.all_reduce(torch.from_numpy(np.ctypeslib.as_array(buf, shape=(int(n),))), group=group)
                return 0
            except Exception as e:  # pragma: no cover
                print("HostComm allreduce failed:", e)
                return 1

        self._cb = (_EXCHANGE_FN(exchange), _ALLREDUCE_FN(allreduce))   # keep the trampolines alive
        h = ctypes.c_void_p()
        _chk(_lib.hhg_comm_create_host(int(self.world), int(self.rank), ctypes.cast(self._cb[0], ctypes.c_void_p),
                                       ctypes.cast(self._cb[1], ctypes.c_void_p), None, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_comm_destroy(self.handle)
            self.handle = None


def icoshell_macro(ntan, nrad, r_min=0.55, r_max=1.0):
    """hhg_icoshell_macro: (verts (V,3), tets (T,4) int32, vtag (V,) int32) of shell(ntan, nrad)."""
    nv, nt = ctypes.c_int64(), ctypes.c_int64()
    _chk(_lib.hhg_icoshell_macro(int(ntan), int(nrad), float(r_min), float(r_max), None, None, None,
                                 ctypes.byref(nv), ctypes.byref(nt)))
    v = np.empty((nv.value, 3), dtype=np.float64)
    t = np.empty((nt.value, 4), dtype=np.int32)
    g = np.empty(nv.value, dtype=np.int32)
    _chk(_lib.hhg_icoshell_macro(int(ntan), int(nrad), float(r_min), float(r_max), _ptr(v), _ptr(t), _ptr(g), None, None))
    return v, t, g


def partition_rcb(verts, tets, nparts, radial=True):
    """hhg_partition_rcb: recursive coordinate bisection of macro centroids (projected to the unit
    sphere when radial, keeping radial macro columns together) -> tet_rank (int32)."""
    v = np.ascontiguousarray(verts, dtype=np.float64)
    t = np.ascontiguousarray(tets, dtype=np.int32)
    out = np.empty(t.shape[0], dtype=np.int32)
    _chk(_lib.hhg_partition_rcb(_ptr(v), v.shape[0], _ptr(t), t.shape[0], int(nparts), 1 if radial else 0,
                                _ptr(out)))
    return out


class Mesh:
    """hhg_mesh_create + blend_map + hhg_set_bc (macro tets uniformly refined to level_max).
    With comm (+ tet_rank) this process keeps its own macros and interface sums / dots run over NCCL;
    ``Mesh.part`` builds rank `rank`'s view of a partition without a communicator (split-phase
    exchange through halo_pack / interface_sum_remote, e.g. several partitions on one GPU)."""

    def __init__(self, verts, tets, vtag=None, level_max=4, tet_rank=None, comm=None, part=None):
        v = np.ascontiguousarray(verts, dtype=np.float64)
        t = np.ascontiguousarray(tets, dtype=np.int32)
        g = None if vtag is None else np.ascontiguousarray(vtag, dtype=np.int32)
        r = None if tet_rank is None else np.ascontiguousarray(tet_rank, dtype=np.int32)
        h = ctypes.c_void_p()
        if part is not None:
            nranks, rank = part
            _chk(_lib.hhg_mesh_create_part(_ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(g), int(level_max), _ptr(r),
                                           int(nranks), int(rank), ctypes.byref(h)))
        else:
            _chk(_lib.hhg_mesh_create(_ptr(v), v.shape[0], _ptr(t), t.shape[0], _ptr(g), int(level_max), _ptr(r),
                                      None if comm is None else comm.handle, ctypes.byref(h)))
        self.handle = h
        self.level_max = level_max
        self.comm = comm

    @classmethod
    def part(cls, macro, level_max, tet_rank, nranks, rank):
        return cls(macro.verts, macro.tets, macro.vtag, level_max, tet_rank=tet_rank, part=(nranks, rank))

    def rank(self):
        r, n = ctypes.c_int(), ctypes.c_int()
        _chk(_lib.hhg_mesh_rank(self.handle, ctypes.byref(r), ctypes.byref(n)))
        return r.value, n.value

    def halo_info(self, level, space):
        """(neighbor ranks, shared-node counts) of the cross-rank interface (host-only)."""
        n = ctypes.c_int()
        _chk(_lib.hhg_halo_info(self.handle, level, space, ctypes.byref(n), None, None))
        nb = np.empty(n.value, dtype=np.int32)
        cnt = np.empty(n.value, dtype=np.int64)
        _chk(_lib.hhg_halo_info(self.handle, level, space, ctypes.byref(n), _ptr(nb), _ptr(cnt)))
        return nb, cnt

    def halo_keys(self, level, space):
        nb, cnt = self.halo_info(level, space)
        keys = np.empty((int(cnt.sum()), 10), dtype=np.int64)
        _chk(_lib.hhg_halo_keys(self.handle, level, space, _ptr(keys)))
        return keys

    def owned_count(self, level, space):
        n = ctypes.c_int64()
        _chk(_lib.hhg_owned_count(self.handle, level, space, ctypes.byref(n)))
        return n.value

    def halo_pack(self, level, space, v, sendbuf=None, stream=None):
        import torch
        nb, cnt = self.halo_info(level, space)
        nc = 3 if space == HHG_P2VEC else 1
        sendbuf = torch.zeros(max(1, int(cnt.sum()) * nc), dtype=torch.float64, device="cuda") \
            if sendbuf is None else sendbuf
        _chk(_lib.hhg_halo_pack(self.handle, level, space, _dev(v, self.vec_len(level, space)), _dev(sendbuf),
                                _stream(stream)))
        return sendbuf

    def interface_sum_remote(self, level, space, recvbuf, v, stream=None):
        _chk(_lib.hhg_interface_sum_remote(self.handle, level, space, _dev(recvbuf),
                                           _dev(v, self.vec_len(level, space)), _stream(stream)))
        return v

    @classmethod
    def from_macro(cls, macro, level_max, **kw):
        return cls(macro.verts, macro.tets, macro.vtag, level_max, **kw)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_mesh_destroy(self.handle)
            self.handle = None

    def set_deterministic(self, on=True):
        """hhg_set_deterministic: colour-ordered element kernels without fp64 atomics (bitwise
        reproducible results; slower)."""
        _chk(_lib.hhg_set_deterministic(self.handle, 1 if on else 0))
        return self

    def prepare(self):
        """hhg_mesh_prepare: build every level's tables now (never lazily in a later call)."""
        _chk(_lib.hhg_mesh_prepare(self.handle))
        return self

    def blend_map(self, kind=HHG_BLEND_SHELL):
        _chk(_lib.blend_map(self.handle, kind))
        return self

    def set_bc(self, tag, kind):
        _chk(_lib.hhg_set_bc(self.handle, tag, kind))
        return self

    def vec_len(self, level, space):
        n = ctypes.c_int64()
        _chk(_lib.hhg_vec_len(self.handle, level, space, ctypes.byref(n)))
        return n.value

    def canonical_len(self, level, space):
        n = ctypes.c_int64()
        _chk(_lib.hhg_canonical_len(self.handle, level, space, ctypes.byref(n)))
        return n.value

    def canonical_keys(self, level, space):
        n = self.canonical_len(level, space)
        keys = np.empty((n, 10), dtype=np.int64)
        _chk(_lib.hhg_canonical_keys(self.handle, level, space, _ptr(keys)))
        return keys

    def zeros(self, level, space):
        import torch
        return torch.zeros(self.vec_len(level, space), dtype=torch.float64, device="cuda")

    def to_canonical(self, level, space, v, stream=None):
        import torch
        out = torch.zeros(self.canonical_len(level, space), dtype=torch.float64, device="cuda")
        _chk(_lib.hhg_to_canonical(self.handle, level, space, _dev(v, self.vec_len(level, space)), _dev(out),
                                   _stream(stream)))
        return out

    def from_canonical(self, level, space, c, stream=None):
        import torch
        c = torch.as_tensor(c, dtype=torch.float64).cuda().contiguous()
        out = self.zeros(level, space)
        _chk(_lib.hhg_from_canonical(self.handle, level, space, _dev(c, self.canonical_len(level, space)),
                                     _dev(out), _stream(stream)))
        return out

    def node_coords(self, level, space, stream=None):
        import torch
        n = self.vec_len(level, space)
        out = torch.empty((n, 3), dtype=torch.float64, device="cuda")
        _chk(_lib.hhg_node_coords(self.handle, level, space, _dev(out), _stream(stream)))
        return out

    def apply_bc(self, level, u, stream=None):
        _chk(_lib.hhg_apply_bc(self.handle, level, _dev(u, self.vec_len(level, HHG_P2VEC)), _stream(stream)))
        return u

    def interface_sum(self, level, space, v, stream=None):
        _chk(_lib.hhg_interface_sum(self.handle, level, space, _dev(v, self.vec_len(level, space)), _stream(stream)))
        return v

    def local_macros(self):
        n = ctypes.c_int64()
        _chk(_lib.hhg_mesh_local_macros(self.handle, ctypes.byref(n)))
        return n.value


def epsilon_apply(mesh, level, eta, u, y=None, form=HHG_VISC_FULL, stream=None):
    n = mesh.vec_len(level, HHG_P2VEC)
    y = mesh.zeros(level, HHG_P2VEC) if y is None else y
    _chk(_lib.epsilon_apply(mesh.handle, level, form, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"),
                            _dev(u, n, "u"), _dev(y, n, "y"), _stream(stream)))
    return y


def epsilon_apply_partial(mesh, level, eta, u, y=None, form=HHG_VISC_FULL, stream=None):
    """Element contributions only (per-copy partial sums, no interface sum, no BC)."""
    n = mesh.vec_len(level, HHG_P2VEC)
    y = mesh.zeros(level, HHG_P2VEC) if y is None else y
    _chk(_lib.epsilon_apply_partial(mesh.handle, level, form, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"),
                                    _dev(u, n, "u"), _dev(y, n, "y"), _stream(stream)))
    return y


def hhg_mass_apply(mesh, level, eta, p, y=None, stream=None):
    """y = M_{1/eta} p (eq:schurMass), consistent P1."""
    n1 = mesh.vec_len(level, HHG_P1)
    y = mesh.zeros(level, HHG_P1) if y is None else y
    _chk(_lib.hhg_mass_apply(mesh.handle, level, _dev(eta, n1, "eta"), _dev(p, n1, "p"), _dev(y, n1, "y"),
                             _stream(stream)))
    return y


def hhg_buoyancy_load(mesh, level, T, f=None, stream=None):
    """f = (M P_v) int (T - 1/2)(x/|x|) . phi  (config-4 buoyancy rhs), T a consistent P1 temperature."""
    f = mesh.zeros(level, HHG_P2VEC) if f is None else f
    _chk(_lib.hhg_buoyancy_load(mesh.handle, level, _dev(T, mesh.vec_len(level, HHG_P1), "T"),
                                _dev(f, mesh.vec_len(level, HHG_P2VEC), "f"), _stream(stream)))
    return f


def hhg_mass_diag(mesh, level, eta, out=None, stream=None):
    n1 = mesh.vec_len(level, HHG_P1)
    out = mesh.zeros(level, HHG_P1) if out is None else out
    _chk(_lib.hhg_mass_diag(mesh.handle, level, _dev(eta, n1, "eta"), _dev(out, n1), _stream(stream)))
    return out


def hhg_kp1_apply(mesh, level, eta, a, p, y=None, stream=None):
    """y = K_{1/sqrt(eta_a)} p: P1 Laplacian weighted by 1/sqrt(eta_a), eta_a = a^2 eta on D_eta (w-BFBT)."""
    n1 = mesh.vec_len(level, HHG_P1)
    y = mesh.zeros(level, HHG_P1) if y is None else y
    _chk(_lib.hhg_kp1_apply(mesh.handle, level, _dev(eta, n1, "eta"), float(a), _dev(p, n1, "p"), _dev(y, n1, "y"),
                            _stream(stream)))
    return y


def hhg_kp1_diag(mesh, level, eta, a, out=None, stream=None):
    n1 = mesh.vec_len(level, HHG_P1)
    out = mesh.zeros(level, HHG_P1) if out is None else out
    _chk(_lib.hhg_kp1_diag(mesh.handle, level, _dev(eta, n1, "eta"), float(a), _dev(out, n1), _stream(stream)))
    return out


def hhg_vmass_apply(mesh, level, eta, a, u, y=None, stream=None):
    """y = (M P_v) M_{sqrt(eta_a)} u: P2 vector mass weighted by sqrt(eta_a) (w-BFBT)."""
    n = mesh.vec_len(level, HHG_P2VEC)
    y = mesh.zeros(level, HHG_P2VEC) if y is None else y
    _chk(_lib.hhg_vmass_apply(mesh.handle, level, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"), float(a),
                              _dev(u, n, "u"), _dev(y, n, "y"), _stream(stream)))
    return y


def hhg_vmass_diag(mesh, level, eta, a, out=None, stream=None):
    n = mesh.vec_len(level, HHG_P2VEC)
    out = mesh.zeros(level, HHG_P2VEC) if out is None else out
    _chk(_lib.hhg_vmass_diag(mesh.handle, level, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"), float(a),
                             _dev(out, n), _stream(stream)))
    return out


def p1_prolong(mesh, coarse_level, x_coarse, x_fine, stream=None):
    """x_fine += P x_coarse (P1 linear interpolation)."""
    _chk(_lib.p1_prolong(mesh.handle, coarse_level, _dev(x_coarse, mesh.vec_len(coarse_level, HHG_P1)),
                         _dev(x_fine, mesh.vec_len(coarse_level + 1, HHG_P1)), _stream(stream)))
    return x_fine


def p1_restrict(mesh, fine_level, r_fine, r_coarse=None, stream=None):
    r_coarse = mesh.zeros(fine_level - 1, HHG_P1) if r_coarse is None else r_coarse
    _chk(_lib.p1_restrict(mesh.handle, fine_level, _dev(r_fine, mesh.vec_len(fine_level, HHG_P1)),
                          _dev(r_coarse, mesh.vec_len(fine_level - 1, HHG_P1)), _stream(stream)))
    return r_coarse


def epsilon_apply_qeta(mesh, level, T2, qeta, u, y=None, stream=None):
    """y = (M P_v) A(eta) u with eta_q = exp(lnC (1/2 - T_q)) (jump if r_q < r_jump else 1) at the
    quadrature points, T_q the P2 interpolant of T2 (NEXT-2 tier); qeta = (lnC, jump, r_jump)."""
    n = mesh.vec_len(level, HHG_P2VEC)
    y = mesh.zeros(level, HHG_P2VEC) if y is None else y
    _chk(_lib.epsilon_apply_qeta(mesh.handle, level, _dev(T2, mesh.vec_len(level, HHG_P2), "T2"), *[float(v) for v in qeta],
                                 _dev(u, n, "u"), _dev(y, n, "y"), _stream(stream)))
    return y


def hhg_diag_qeta(mesh, level, T2, qeta, out=None, stream=None):
    out = mesh.zeros(level, HHG_P2VEC) if out is None else out
    _chk(_lib.hhg_diag_qeta(mesh.handle, level, _dev(T2, mesh.vec_len(level, HHG_P2), "T2"), *[float(v) for v in qeta],
                            _dev(out, mesh.vec_len(level, HHG_P2VEC)), _stream(stream)))
    return out


def div_apply(mesh, level, gamma, u, q=None, stream=None):
    q = mesh.zeros(level, HHG_P1) if q is None else q
    _chk(_lib.div_apply(mesh.handle, level, float(gamma), _dev(u, mesh.vec_len(level, HHG_P2VEC), "u"),
                        _dev(q, mesh.vec_len(level, HHG_P1), "q"), _stream(stream)))
    return q


def divT_apply(mesh, level, p, y=None, accumulate=False, stream=None):
    y = mesh.zeros(level, HHG_P2VEC) if y is None else y
    _chk(_lib.divT_apply(mesh.handle, level, _dev(p, mesh.vec_len(level, HHG_P1), "p"),
                         _dev(y, mesh.vec_len(level, HHG_P2VEC), "y"), 1 if accumulate else 0, _stream(stream)))
    return y


def stokes_apply(mesh, level, eta, gamma, u, p, y_u=None, y_p=None, stream=None):
    y_u = mesh.zeros(level, HHG_P2VEC) if y_u is None else y_u
    y_p = mesh.zeros(level, HHG_P1) if y_p is None else y_p
    n2, n1 = mesh.vec_len(level, HHG_P2VEC), mesh.vec_len(level, HHG_P1)
    _chk(_lib.stokes_apply(mesh.handle, level, _dev(eta, n1, "eta"), float(gamma), _dev(u, n2, "u"), _dev(p, n1, "p"),
                           _dev(y_u, n2, "y_u"), _dev(y_p, n1, "y_p"), _stream(stream)))
    return y_u, y_p


def hhg_diag(mesh, level, eta, out=None, stream=None):
    out = mesh.zeros(level, HHG_P2VEC) if out is None else out
    _chk(_lib.hhg_diag(mesh.handle, level, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"),
                       _dev(out, mesh.vec_len(level, HHG_P2VEC)), _stream(stream)))
    return out


def hhg_dot(mesh, level, space, x, y, stream=None):
    import torch
    out = torch.zeros(1, dtype=torch.float64, device="cuda")
    n = mesh.vec_len(level, space)
    _chk(_lib.hhg_dot(mesh.handle, level, space, _dev(x, n), _dev(y, n), _dev(out), _stream(stream)))
    return out


def p2_restrict(mesh, fine_level, r_fine, r_coarse=None, stream=None):
    r_coarse = mesh.zeros(fine_level - 1, HHG_P2VEC) if r_coarse is None else r_coarse
    _chk(_lib.p2_restrict(mesh.handle, fine_level, _dev(r_fine, mesh.vec_len(fine_level, HHG_P2VEC)),
                          _dev(r_coarse, mesh.vec_len(fine_level - 1, HHG_P2VEC)), _stream(stream)))
    return r_coarse


def p2_prolong(mesh, coarse_level, x_coarse, x_fine, stream=None):
    _chk(_lib.p2_prolong(mesh.handle, coarse_level, _dev(x_coarse, mesh.vec_len(coarse_level, HHG_P2VEC)),
                         _dev(x_fine, mesh.vec_len(coarse_level + 1, HHG_P2VEC)), _stream(stream)))
    return x_fine


def chebyshev_smooth(mesh, level, eta, dinv, degree, lmin, lmax, rhs, x, work=None, stream=None):
    import torch
    n = mesh.vec_len(level, HHG_P2VEC)
    work = torch.empty(3 * n, dtype=torch.float64, device="cuda") if work is None else work
    _chk(_lib.chebyshev_smooth(mesh.handle, level, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"), _dev(dinv, n),
                               int(degree), float(lmin), float(lmax), _dev(rhs, n), _dev(x, n), _dev(work),
                               _stream(stream)))
    return x


def hhg_power_iteration(mesh, level, eta, dinv, iters, v0, stream=None):
    n = mesh.vec_len(level, HHG_P2VEC)
    lam = ctypes.c_double()
    _chk(_lib.hhg_power_iteration(mesh.handle, level, _dev(eta, mesh.vec_len(level, HHG_P1), "eta"), _dev(dinv, n),
                                  int(iters), _dev(v0, n), ctypes.byref(lam), _stream(stream)))
    return lam.value


class _MGParams(ctypes.Structure):
    _fields_ = [("l_min", ctypes.c_int), ("l_max", ctypes.c_int), ("pre", ctypes.c_int), ("post", ctypes.c_int),
                ("degree", ctypes.c_int), ("power_iters", ctypes.c_int), ("coarse_iters", ctypes.c_int),
                ("cheb_hi_factor", ctypes.c_double), ("cheb_lo_ratio", ctypes.c_double),
                ("visc_form", ctypes.c_int), ("use_graph", ctypes.c_int), ("l_eta", ctypes.c_int),
                ("qeta_lnC", ctypes.c_double), ("qeta_jump", ctypes.c_double), ("qeta_rjump", ctypes.c_double),
                ("coarse_redundant", ctypes.c_int), ("coarse_tol", ctypes.c_double)]


class MG:
    """hhg_mg_create: per-level D^-1 and lambda_hat; vcycle() applies one V-cycle."""

    def __init__(self, mesh, l_min, l_max, eta_per_level, power_v0, pre=3, post=3, degree=3, power_iters=20,
                 coarse_iters=50, hi=1.1, lo=0.1, form=HHG_VISC_FULL, use_graph=True, T2_per_level=None, l_eta=-1,
                 qeta=(0.0, 1.0, 0.0), coarse_redundant=True, coarse_tol=0.0):
        """T2_per_level / l_eta / qeta = (lnC, jump, r_jump): on levels <= l_eta the viscosity is evaluated
        at the quadrature points from the P2 temperature (NEXT-2 tier).  coarse_redundant
        (multi-rank meshes): solve the gathered coarse problem on every rank.  coarse_tol > 0:
        the coarse PCG stops at sqrt(r.z) <= coarse_tol sqrt(r0.z0), at most coarse_iters (Table 1)."""
        self.mesh = mesh
        self.l_min, self.l_max = l_min, l_max
        prm = _MGParams(l_min, l_max, pre, post, degree, power_iters, coarse_iters, hi, lo, form,
                        1 if use_graph else 0, int(l_eta), *[float(v) for v in qeta], 1 if coarse_redundant else 0,
                        float(coarse_tol))
        self._eta = dict(eta_per_level)
        self._v0 = dict(power_v0)
        self._T2 = dict(T2_per_level or {})
        L = l_max + 1
        etas = (ctypes.c_void_p * L)(*[_ptr(self._eta.get(l)) for l in range(L)])
        v0s = (ctypes.c_void_p * L)(*[_ptr(self._v0.get(l)) for l in range(L)])
        h = ctypes.c_void_p()
        if T2_per_level:
            t2 = (ctypes.c_void_p * L)(*[_ptr(self._T2.get(l)) for l in range(L)])
            _chk(_lib.hhg_mg_create_qeta(mesh.handle, ctypes.byref(prm), etas, t2, v0s, ctypes.byref(h)))
        else:
            _chk(_lib.hhg_mg_create(mesh.handle, ctypes.byref(prm), etas, v0s, ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_mg_destroy(self.handle)
            self.handle = None

    def lam(self, level):
        v = ctypes.c_double()
        _chk(_lib.hhg_mg_lambda(self.handle, level, ctypes.byref(v)))
        return v.value

    def coarse_iterations(self):
        """iterations of the most recent coarse solve (synchronises)"""
        v = ctypes.c_int()
        _chk(_lib.hhg_mg_coarse_iterations(self.handle, ctypes.byref(v)))
        return v.value

    def vcycle(self, rhs, x=None, stream=None):
        n = self.mesh.vec_len(self.l_max, HHG_P2VEC)
        x = self.mesh.zeros(self.l_max, HHG_P2VEC) if x is None else x
        _chk(_lib.vcycle(self.handle, _dev(rhs, n, "rhs"), _dev(x, n, "x"), _stream(stream)))
        return x

    def ablock_cg(self, rhs, x=None, tol=1e-2, max_iters=100, stream=None):
        """A-block CG preconditioned by this V-cycle -> (x, iterations, relative residual)."""
        n = self.mesh.vec_len(self.l_max, HHG_P2VEC)
        x = self.mesh.zeros(self.l_max, HHG_P2VEC) if x is None else x
        it, rel = ctypes.c_int(), ctypes.c_double()
        _chk(_lib.hhg_ablock_cg(self.handle, _dev(rhs, n, "rhs"), _dev(x, n, "x"), float(tol), int(max_iters),
                                ctypes.byref(it), ctypes.byref(rel), _stream(stream)))
        return x, it.value, rel.value

    def _host_vec(self, t, name):
        import torch
        n = self.mesh.vec_len(self.l_max, HHG_P2VEC)
        if not (isinstance(t, torch.Tensor) and t.device.type == "cpu" and t.dtype == torch.float64
                and t.is_contiguous() and t.numel() == n):
            raise HHGError(f"{name}: need a contiguous float64 host tensor of length {n}")
        return t

    def vcycle_host(self, rhs_host, x_host, stream=None):
        """One V-cycle on host buffers (H2D, V-cycle, D2H on `stream`; asynchronous when the buffers
        are pinned -- the binding keeps references to them until the next call)."""
        self._host_vec(rhs_host, "rhs_host")
        self._host_vec(x_host, "x_host")
        self._host_keep = (rhs_host, x_host)
        _chk(_lib.vcycle_host(self.handle, _ptr(rhs_host), _ptr(x_host), _stream(stream)))
        return x_host

    def vcycle_host_batch(self, rhs_hosts, x_hosts, stream=None):
        """One V-cycle per (rhs_hosts[k] -> x_hosts[k]) pair of pinned host tensors, with the copies of
        neighbouring steps overlapped with the compute (asynchronous on `stream`)."""
        k = len(rhs_hosts)
        assert len(x_hosts) == k
        for t in list(rhs_hosts) + list(x_hosts):
            self._host_vec(t, "vcycle_host_batch")
            if not t.is_pinned():
                raise HHGError("vcycle_host_batch: need pinned host tensors")
        self._batch_keep = (list(rhs_hosts), list(x_hosts))
        rh = (ctypes.c_void_p * k)(*[t.data_ptr() for t in rhs_hosts])
        xh = (ctypes.c_void_p * k)(*[t.data_ptr() for t in x_hosts])
        _chk(_lib.vcycle_host_batch(self.handle, rh, xh, k, _stream(stream)))
        return x_hosts

    def profile(self, enable=True):
        _chk(_lib.hhg_mg_profile(self.handle, 1 if enable else 0))

    def profile_get(self):
        a, c = ctypes.c_double(), ctypes.c_double()
        na, nc = ctypes.c_int64(), ctypes.c_int64()
        _chk(_lib.hhg_mg_profile_get(self.handle, ctypes.byref(a), ctypes.byref(na), ctypes.byref(c),
                                     ctypes.byref(nc)))
        d = ctypes.c_double()
        _chk(_lib.hhg_mg_profile_get_dense(self.handle, ctypes.byref(d)))
        return dict(apply_ms_sum=a.value, apply_count=na.value, cycle_ms_sum=c.value, cycle_count=nc.value,
                    dense_ms_sum=d.value)


class KMG:
    """hhg_kmg_create: GMG-preconditioned CG for K_{1/sqrt(eta_a)} (the w-BFBT Poisson solve)."""

    def __init__(self, mesh, l_min, l_max, eta_per_level, a=1.0, pre=3, post=3, degree=3, power_iters=20,
                 coarse_iters=50, hi=1.1, lo=0.1):
        self.mesh, self.l_min, self.l_max = mesh, l_min, l_max
        prm = _MGParams(l_min, l_max, pre, post, degree, power_iters, coarse_iters, hi, lo, HHG_VISC_FULL, 0, -1,
                        0.0, 1.0, 0.0, 0)
        self._eta = dict(eta_per_level or {})
        L = l_max + 1
        etas = (ctypes.c_void_p * L)(*[_ptr(self._eta.get(l)) for l in range(L)])
        h = ctypes.c_void_p()
        _chk(_lib.hhg_kmg_create(mesh.handle, ctypes.byref(prm), etas, float(a), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_kmg_destroy(self.handle)
            self.handle = None

    def solve(self, rhs, x=None, tol=1e-8, tol_abs=0.0, max_iters=100, stream=None):
        n = self.mesh.vec_len(self.l_max, HHG_P1)
        x = self.mesh.zeros(self.l_max, HHG_P1) if x is None else x
        it, rel = ctypes.c_int(), ctypes.c_double()
        _chk(_lib.hhg_kmg_solve(self.handle, _dev(rhs, n, "rhs"), _dev(x, n, "x"), float(tol), float(tol_abs),
                                int(max_iters), ctypes.byref(it), ctypes.byref(rel), _stream(stream)))
        return x, it.value, rel.value


class _TempParams(ctypes.Structure):
    _fields_ = [("s", ctypes.c_double), ("tau", ctypes.c_double), ("kappa", ctypes.c_double),
                ("beta", ctypes.c_double), ("gamma", ctypes.c_double)]


def hhg_temp_apply(mesh, level, prm, u, T, y=None, which=0, stream=None):
    """y = L T (which 0), P T (1) or diag P (2) of eq:WeakTemp; prm = dict(s, tau, kappa, beta, gamma)."""
    n = mesh.vec_len(level, HHG_P2)
    y = mesh.zeros(level, HHG_P2) if y is None else y
    p = _TempParams(**{k: float(v) for k, v in prm.items()})
    _chk(_lib.hhg_temp_apply(mesh.handle, level, ctypes.byref(p), _dev(u, mesh.vec_len(level, HHG_P2VEC), "u"),
                             _dev(T, n, "T"), _dev(y, n, "y"), int(which), _stream(stream)))
    return y


def hhg_mmoc(mesh, level, T, u_new, u_old, tau, T_hat=None, stream=None):
    """T_hat = T at the RK4 back-tracked positions of the P2 nodes (MMOC)."""
    n = mesh.vec_len(level, HHG_P2)
    nv = mesh.vec_len(level, HHG_P2VEC)
    T_hat = mesh.zeros(level, HHG_P2) if T_hat is None else T_hat
    _chk(_lib.hhg_mmoc(mesh.handle, level, _dev(T, n, "T"), _dev(u_new, nv, "u_new"), _dev(u_old, nv, "u_old"),
                       float(tau), _dev(T_hat, n, "T_hat"), _stream(stream)))
    return T_hat


class TempSolver:
    """hhg_temp_solver_*: FGMRES preconditioned by CG on the mass + diffusion part."""

    def __init__(self, mesh, level, prm, restart=30):
        self.mesh, self.level = mesh, level
        p = _TempParams(**{k: float(v) for k, v in prm.items()})
        h = ctypes.c_void_p()
        _chk(_lib.hhg_temp_solver_create(mesh.handle, level, ctypes.byref(p), int(restart), ctypes.byref(h)))
        self.handle = h

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_temp_solver_destroy(self.handle)
            self.handle = None

    def solve(self, u, b, T, tol=1e-10, tol_abs=0.0, max_iters=100, tol_cg=1e-13, cg_max_iters=2000, stream=None):
        """T: in = Dirichlet values on the boundary nodes, out = solution -> (T, iterations, rel. residual)."""
        n = self.mesh.vec_len(self.level, HHG_P2)
        it, rel = ctypes.c_int(), ctypes.c_double()
        _chk(_lib.hhg_temp_solve(self.handle, _dev(u, self.mesh.vec_len(self.level, HHG_P2VEC), "u"), _dev(b, n, "b"),
                                 _dev(T, n, "T"), float(tol), float(tol_abs), int(max_iters), float(tol_cg),
                                 int(cg_max_iters), ctypes.byref(it), ctypes.byref(rel), _stream(stream)))
        return T, it.value, rel.value


class _StokesParams(ctypes.Structure):
    _fields_ = [("restart", ctypes.c_int), ("max_iters", ctypes.c_int), ("tol", ctypes.c_double),
                ("sigma", ctypes.c_double), ("omega", ctypes.c_double), ("tol_A", ctypes.c_double),
                ("ablock_max_iters", ctypes.c_int), ("tol_mass", ctypes.c_double), ("mass_max_iters", ctypes.c_int),
                ("schur", ctypes.c_int), ("tol_vbfbt", ctypes.c_double), ("vbfbt_max_iters", ctypes.c_int),
                ("uzawa", ctypes.c_int), ("a_l", ctypes.c_double), ("a_r", ctypes.c_double),
                ("tol_wbfbt", ctypes.c_double), ("tol_wbfbt_abs", ctypes.c_double), ("wbfbt_max_iters", ctypes.c_int),
                ("tol_vmass", ctypes.c_double), ("vmass_max_iters", ctypes.c_int)]


class StokesSolver:
    """hhg_stokes_create / hhg_stokes_solve: FGMRES + symmetric Uzawa (A^-1: V-cycle CG, S^-1: M_{1/eta}
    CG) on the finest level of `mg`.  Vectors are [u (P2VEC) | p (P1)] concatenated."""

    def __init__(self, mg, eta, gamma, restart=30, max_iters=100, tol=1e-8, sigma=1.0, omega=0.3, tol_A=1e-2,
                 ablock_max_iters=200, tol_mass=1e-10, mass_max_iters=500, schur="mass", mg_cheap=None,
                 tol_vbfbt=1e-1, vbfbt_max_iters=100, uzawa="symmetric", a_l=1.0, a_r=1.0, tol_wbfbt=1e-10,
                 tol_wbfbt_abs=1e-10, wbfbt_max_iters=100, tol_vmass=1e-4, vmass_max_iters=500):
        """schur: "mass" (S = M_{1/eta}, eq:schurMass), "vbfbt" (eq:schurV; mg_cheap = the A_C hierarchy,
        Table 1: V(1,1) with degree-1 Chebyshev) or "wbfbt" (eq:schurWBFBT with the a_l / a_r scaling;
        K_{1/sqrt(eta)} by GMG-CG to tol_wbfbt / tol_wbfbt_abs, M_{sqrt(eta)} by Jacobi-CG to tol_vmass;
        defaults from Table 1: 1e-10, 1e-4, a_l = a_r = 1)."""
        self.mg, self.mg_cheap = mg, mg_cheap
        self._eta = eta
        prm = _StokesParams(restart, max_iters, tol, sigma, omega, tol_A, ablock_max_iters, tol_mass, mass_max_iters,
                            {"mass": 0, "vbfbt": 1, "wbfbt": 2}[schur], tol_vbfbt, vbfbt_max_iters,
                            {"symmetric": 0, "inexact": 1, "adjoint": 2}[uzawa], a_l, a_r, tol_wbfbt, tol_wbfbt_abs,
                            wbfbt_max_iters, tol_vmass, vmass_max_iters)
        h = ctypes.c_void_p()
        _chk(_lib.hhg_stokes_create(mg.handle, None if mg_cheap is None else mg_cheap.handle, _ptr(eta), float(gamma),
                                    ctypes.byref(prm), ctypes.byref(h)))
        self.handle = h
        L = mg.l_max
        self.n2, self.n1 = mg.mesh.vec_len(L, HHG_P2VEC), mg.mesh.vec_len(L, HHG_P1)

    def __del__(self):
        if getattr(self, "handle", None) and _lib is not None:
            _lib.hhg_stokes_destroy(self.handle)
            self.handle = None

    def schur_apply(self, t, z=None, stream=None):
        """z = S^-1 t of the solver's Schur approximation (no -omega), mean zero."""
        z = self.mg.mesh.zeros(self.mg.l_max, HHG_P1) if z is None else z
        _chk(_lib.hhg_stokes_schur_apply(self.handle, _dev(t, self.n1, "t"), _dev(z, self.n1, "z"), _stream(stream)))
        return z

    def solve(self, rhs, x=None, stream=None):
        import torch
        n = self.n2 + self.n1
        x = torch.zeros(n, dtype=torch.float64, device="cuda") if x is None else x
        it, rel = ctypes.c_int(), ctypes.c_double()
        _chk(_lib.hhg_stokes_solve(self.handle, _dev(rhs, n, "rhs"), _dev(x, n, "x"), ctypes.byref(it),
                                   ctypes.byref(rel), _stream(stream)))
        return x, it.value, rel.value

