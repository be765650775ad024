"""Thin ctypes binding of the lorpc C ABI (include/lorpc.h).

Argument marshalling only: every step of the hot path runs in the CUDA kernels
of liblorpc.so.  Device vectors are torch CUDA float64 tensors (torch supplies
device memory and streams); host arrays are numpy float64.  There is no CPU
fallback: if liblorpc.so is missing or a call fails, an exception is raised.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liblorpc.so")
_lib = None

_vp = ctypes.c_void_p
_int = ctypes.c_int
_ll = ctypes.c_longlong
_d = ctypes.c_double


class LorpcError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"lorpc error {code}: {msg}")
        self.code = code


class MeshDesc(ctypes.Structure):
    _fields_ = [("dim", _int), ("n", _int * 3), ("p", _int), ("disc", _int), ("eta", _d), ("quad", _int)]


class SchwarzDesc(ctypes.Structure):
    _fields_ = [("patch_kind", _int), ("ordering", _int), ("coarse", _int), ("extend", _int)]


class PcgReport(ctypes.Structure):
    _fields_ = [("iters", _int), ("converged", _int), ("rel_res", _d),
                ("res_hist", ctypes.POINTER(_d)), ("alpha", ctypes.POINTER(_d)),
                ("beta", ctypes.POINTER(_d)), ("t_solve_ms", _d)]


SYMBOLS = ["lorpc_mesh_create", "lorpc_mesh_destroy", "lorpc_mesh_sizes", "lorpc_quad_points",
           "lorpc_rhs_assemble", "lorpc_mesh_set_coefficient", "lorpc_subcell_points", "lorpc_operator_apply", "lorpc_lor_assemble", "lorpc_lor_destroy",
           "lorpc_schwarz_setup", "lorpc_prec_destroy", "lorpc_precond_apply",
           "lorpc_prec_export_ordering", "lorpc_prec_info", "lorpc_prec_kernel", "lorpc_prec_bytes", "lorpc_prec_profile",
           "lorpc_prec_profile_read", "lorpc_pcg_solve", "lorpc_pcg_solve_host",
           "lorpc_launch_count", "lorpc_last_error",
           "lorpc_dist_plan_get", "lorpc_dist_nccl_id", "lorpc_dist_create", "lorpc_dist_destroy",
           "lorpc_dist_info", "lorpc_dist_local_prec", "lorpc_dist_operator_apply", "lorpc_dist_precond_apply", "lorpc_dist_pcg_solve"]


class DistPlan(ctypes.Structure):
    _fields_ = [("z0", _int), ("z1", _int), ("za", _int), ("zb", _int), ("own_plane0", _int),
                ("own_planes", _int), ("gown_plane0", _int), ("vown0", _int), ("nvown", _int),
                ("to", _int * 4), ("from_", _int * 4), ("send0", _int * 4), ("recv0", _int * 4),
                ("nplanes", _int * 4)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run __graft_entry__.build() (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        L.lorpc_last_error.restype = ctypes.c_char_p
        L.lorpc_mesh_create.argtypes = [ctypes.POINTER(MeshDesc), _vp, _vp, ctypes.POINTER(_vp)]
        L.lorpc_mesh_destroy.argtypes = [_vp]
        L.lorpc_mesh_sizes.argtypes = [_vp, ctypes.POINTER(_ll), ctypes.POINTER(_ll), ctypes.POINTER(_ll)]
        L.lorpc_quad_points.argtypes = [_vp, _vp, _vp, _vp]
        L.lorpc_rhs_assemble.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.lorpc_mesh_set_coefficient.argtypes = [_vp, _vp, _vp, _vp]
        L.lorpc_subcell_points.argtypes = [_vp, _vp, ctypes.POINTER(_ll), _vp]
        L.lorpc_operator_apply.argtypes = [_vp, _vp, _vp, _vp]
        L.lorpc_lor_assemble.argtypes = [_vp, _vp, ctypes.POINTER(_vp)]
        L.lorpc_lor_destroy.argtypes = [_vp]
        L.lorpc_schwarz_setup.argtypes = [_vp, ctypes.POINTER(SchwarzDesc), _vp, ctypes.POINTER(_vp)]
        L.lorpc_prec_destroy.argtypes = [_vp]
        L.lorpc_precond_apply.argtypes = [_vp, _vp, _vp, _vp]
        L.lorpc_prec_export_ordering.argtypes = [_vp, _ll, _int, ctypes.POINTER(_int), ctypes.POINTER(_int)]
        L.lorpc_prec_info.argtypes = [_vp, ctypes.POINTER(_ll), ctypes.POINTER(_int)]
        L.lorpc_prec_kernel.argtypes = [_vp, ctypes.POINTER(_int)]
        L.lorpc_prec_bytes.argtypes = [_vp, ctypes.POINTER(_ll), ctypes.POINTER(_ll), ctypes.POINTER(_ll)]
        L.lorpc_prec_profile.argtypes = [_vp, _int]
        L.lorpc_prec_profile_read.argtypes = [_vp, ctypes.POINTER(_d), ctypes.POINTER(_ll)]
        L.lorpc_pcg_solve.argtypes = [_vp, _vp, _vp, _vp, _d, _int, ctypes.POINTER(PcgReport), _vp]
        L.lorpc_pcg_solve_host.argtypes = [_vp, _vp, _vp, _vp, _d, _int, ctypes.POINTER(PcgReport), _vp]
        L.lorpc_launch_count.restype = _ll
        L.lorpc_launch_count.argtypes = [_int]
        L.lorpc_dist_plan_get.argtypes = [_int, _int, _int, _int, ctypes.POINTER(DistPlan)]
        L.lorpc_dist_nccl_id.argtypes = [_vp]
        L.lorpc_dist_create.argtypes = [ctypes.POINTER(MeshDesc), _vp, ctypes.POINTER(SchwarzDesc), _int, _int, _vp,
                                        _vp, ctypes.POINTER(_vp)]
        L.lorpc_dist_destroy.argtypes = [_vp]
        L.lorpc_dist_info.argtypes = [_vp, _int, ctypes.POINTER(_ll), ctypes.POINTER(_ll), ctypes.POINTER(_ll)]
        L.lorpc_dist_local_prec.argtypes = [_vp, _int, ctypes.POINTER(_vp)]
        L.lorpc_dist_operator_apply.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
        L.lorpc_dist_precond_apply.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp)]
        L.lorpc_dist_pcg_solve.argtypes = [_vp, ctypes.POINTER(_vp), ctypes.POINTER(_vp), _d, _int,
                                           ctypes.POINTER(PcgReport)]
        _lib = L
    return _lib


def _check(rc):
    if rc != 0:
        raise LorpcError(rc, lib().lorpc_last_error().decode())


def _stream(stream):
    if stream is not None:
        return stream
    import torch
    return torch.cuda.current_stream().cuda_stream


def _dptr(t):
    if t is None:
        return None
    assert t.is_cuda and t.dtype.is_floating_point and t.element_size() == 8 and t.is_contiguous(), \
        "device vectors must be contiguous CUDA float64 tensors"
    return t.data_ptr()


def launch_count(reset=False):
    return lib().lorpc_launch_count(1 if reset else 0)


class Mesh:
    """lorpc_mesh: Cartesian topology of multilinear tensor-product elements."""

    def __init__(self, dim, n, p, vertices, disc=0, eta=0.0, stream=None, quad=0):
        n = list(n) + [1] * (3 - len(n))
        self.desc = MeshDesc(dim, (_int * 3)(*n[:3]), p, disc, float(eta), int(quad))
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        h = _vp()
        _check(lib().lorpc_mesh_create(ctypes.byref(self.desc), V.ctypes.data, _stream(stream), ctypes.byref(h)))
        self.h = h
        self.dim, self.p, self.disc = dim, p, disc
        a, b, c = _ll(), _ll(), _ll()
        _check(lib().lorpc_mesh_sizes(self.h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        self.n_dof, self.n_quad, self.n_bface_quad = a.value, b.value, c.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lorpc_mesh_destroy(self.h)
            self.h = None

    def quad_points(self, xq=None, xbq=None, stream=None):
        _check(lib().lorpc_quad_points(self.h, _dptr(xq), _dptr(xbq), _stream(stream)))

    def subcell_points(self, xs=None, stream=None):
        """Number of LOR subcells; fills xs [n_sub * 2^d * d] with their Gauss points."""
        n = _ll()
        _check(lib().lorpc_subcell_points(self.h, _dptr(xs) if xs is not None else None, ctypes.byref(n),
                                          _stream(stream)))
        return n.value

    def set_coefficient(self, bq, bsub, stream=None):
        """b(x) at the volume Gauss points / LOR subcell Gauss points (row f3)."""
        _check(lib().lorpc_mesh_set_coefficient(self.h, _dptr(bq) if bq is not None else None,
                                                _dptr(bsub) if bsub is not None else None, _stream(stream)))

    def rhs_assemble(self, fq, gq, b, stream=None):
        _check(lib().lorpc_rhs_assemble(self.h, _dptr(fq), _dptr(gq), _dptr(b), _stream(stream)))

    def apply(self, x, y, stream=None):
        _check(lib().lorpc_operator_apply(self.h, _dptr(x), _dptr(y), _stream(stream)))


class Lor:
    """lorpc_lor: K_h on the GLL-refined mesh and the element-structured hierarchy."""

    def __init__(self, mesh, stream=None):
        self.mesh = mesh
        h = _vp()
        _check(lib().lorpc_lor_assemble(mesh.h, _stream(stream), ctypes.byref(h)))
        self.h = h

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lorpc_lor_destroy(self.h)
            self.h = None


PATCH_KIND = {"vertex": 0, "star": 1, "single": 2}
ORDERING = {"mdf": 0, "natural": 1, "rcm": 2}
COARSE = {"gmg": 0, "none": 1}


class Prec:
    """lorpc_prec: additive Schwarz B (eq:as) or B_DG (eq:dg-as)."""

    def __init__(self, lor, patch_kind="vertex", ordering="mdf", coarse="gmg", stream=None, extend=False):
        self.lor = lor
        self.mesh = lor.mesh
        self.desc = SchwarzDesc(PATCH_KIND[patch_kind], ORDERING[ordering], COARSE[coarse], 1 if extend else 0)
        h = _vp()
        _check(lib().lorpc_schwarz_setup(lor.h, ctypes.byref(self.desc), _stream(stream), ctypes.byref(h)))
        self.h = h
        J, L = _ll(), _int()
        _check(lib().lorpc_prec_info(self.h, ctypes.byref(J), ctypes.byref(L)))
        self.n_patches, self.n_levels = J.value, L.value

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lorpc_prec_destroy(self.h)
            self.h = None

    def apply(self, r, z, stream=None):
        _check(lib().lorpc_precond_apply(self.h, _dptr(r), _dptr(z), _stream(stream)))

    KERNELS = {0: "group-mode patch V-cycle (k_vcycle, every level in shared memory)",
               1: "thread-mode patch V-cycle (k_vt_smooth pre + k_vt_mid + k_vt_smooth post)",
               2: "W-mode fused patch V-cycle (k_vw, factor staged in shared memory)",
               3: "thread-mode patch V-cycle, one sweep schedule per warp (U-records: k_vt_smooth pre + k_vt_mid3l / k_vt_mid + k_vt_smooth post)",
               4: "Q-mode fused patch V-cycle (k_vq: LP lanes per patch, factors streamed through a cp.async ring)"}

    def kernel(self):
        """Label of the patch V-cycle kernel family this preconditioner runs."""
        m = _int()
        _check(lib().lorpc_prec_kernel(self.h, ctypes.byref(m)))
        return self.KERNELS[m.value]

    def byte_model(self):
        """(factor values, [level-l grid nodes], coarse GMG nodes) for the roofline model."""
        fv, cn = _ll(), _ll()
        ln = (_ll * 8)()
        _check(lib().lorpc_prec_bytes(self.h, ctypes.byref(fv), ln, ctypes.byref(cn)))
        return fv.value, [ln[i] for i in range(self.n_levels)], cn.value

    def profile(self, enable):
        _check(lib().lorpc_prec_profile(self.h, 1 if enable else 0))

    def profile_read(self):
        ms, n = _d(), _ll()
        _check(lib().lorpc_prec_profile_read(self.h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    def ordering(self, patch, level, cap=1024):
        buf = (_int * cap)()
        n = _int(cap)
        _check(lib().lorpc_prec_export_ordering(self.h, patch, level, buf, ctypes.byref(n)))
        return np.array(buf[:n.value], dtype=np.int64)


def _report(rep, maxit, keep):
    return {"iters": rep.iters, "converged": bool(rep.converged), "rel_res": rep.rel_res,
            "t_solve_ms": rep.t_solve_ms,
            "res": keep[0][:rep.iters + 1].copy(), "alpha": keep[1][:rep.iters].copy(),
            "beta": keep[2][:max(rep.iters - 1, 0)].copy()}


def _mkrep(maxit):
    keep = (np.zeros(maxit + 1), np.zeros(maxit), np.zeros(maxit))
    rep = PcgReport(0, 0, 0.0, keep[0].ctypes.data_as(ctypes.POINTER(_d)),
                    keep[1].ctypes.data_as(ctypes.POINTER(_d)), keep[2].ctypes.data_as(ctypes.POINTER(_d)), 0.0)
    return rep, keep


def pcg_solve(mesh, prec, b, x, rtol, maxit=2000, stream=None, allow_not_converged=False):
    rep, keep = _mkrep(maxit)
    rc = lib().lorpc_pcg_solve(mesh.h, prec.h, _dptr(b), _dptr(x), float(rtol), int(maxit), ctypes.byref(rep),
                               _stream(stream))
    if rc != 0 and not (allow_not_converged and rc == 6):
        _check(rc)
    return _report(rep, maxit, keep)


def pcg_solve_host(mesh, prec, b_host, x_host, rtol, maxit=2000, stream=None):
    """End-to-end solve through the C ABI with host buffers (H2D / D2H inside the call)."""
    rep, keep = _mkrep(maxit)
    b_host = np.ascontiguousarray(b_host, dtype=np.float64)
    assert x_host.dtype == np.float64 and x_host.flags.c_contiguous
    _check(lib().lorpc_pcg_solve_host(mesh.h, prec.h, b_host.ctypes.data, x_host.ctypes.data, float(rtol),
                                      int(maxit), ctypes.byref(rep), _stream(stream)))
    return _report(rep, maxit, keep)


# ---------------------------------------------------------------- multi-GPU slabs
def dist_plan(n_z, p, nranks, rank):
    """Slab plan of one rank (host-only C call): ownership and the four exchange phases."""
    P = DistPlan()
    _check(lib().lorpc_dist_plan_get(int(n_z), int(p), int(nranks), int(rank), ctypes.byref(P)))
    return {"z0": P.z0, "z1": P.z1, "za": P.za, "zb": P.zb, "own_plane0": P.own_plane0,
            "own_planes": P.own_planes, "gown_plane0": P.gown_plane0, "vown0": P.vown0, "nvown": P.nvown,
            "to": list(P.to), "from": list(P.from_), "send0": list(P.send0), "recv0": list(P.recv0),
            "nplanes": list(P.nplanes)}


def dist_nccl_id():
    buf = (ctypes.c_ubyte * 128)()
    _check(lib().lorpc_dist_nccl_id(ctypes.cast(buf, _vp)))
    return bytes(buf)


class Dist:
    """lorpc_dist: the C5-style slab decomposition of the 3D CG path.

    nccl_id=None: all `nranks` ranks emulated in this process on the current device
    (exchanges by device copies); otherwise this process is rank `rank` of an NCCL
    communicator."""

    def __init__(self, n, p, vertices, nranks, rank=0, nccl_id=None, patch_kind="vertex", ordering="mdf",
                 stream=None):
        self.desc = MeshDesc(3, (_int * 3)(*n), p, 0, 0.0, 0)
        self.sdesc = SchwarzDesc(PATCH_KIND[patch_kind], ORDERING[ordering], 0, 0)
        V = np.ascontiguousarray(vertices, dtype=np.float64)
        self._id = (ctypes.c_ubyte * 128)(*nccl_id) if nccl_id is not None else None
        h = _vp()
        _check(lib().lorpc_dist_create(ctypes.byref(self.desc), V.ctypes.data, ctypes.byref(self.sdesc),
                                       int(nranks), int(rank), ctypes.cast(self._id, _vp) if self._id else None,
                                       _stream(stream), ctypes.byref(h)))
        self.h = h
        self.nranks = nranks
        self.nlocal = nranks if nccl_id is None else 1
        self.owned = []
        for i in range(self.nlocal):
            off, cnt, J = _ll(), _ll(), _ll()
            _check(lib().lorpc_dist_info(self.h, i, ctypes.byref(off), ctypes.byref(cnt), ctypes.byref(J)))
            self.owned.append((off.value, cnt.value, J.value))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.lorpc_dist_destroy(self.h)
            self.h = None

    @staticmethod
    def _ptrs(ts):
        return (_vp * len(ts))(*[_dptr(t) for t in ts])

    def local_byte_model(self, local=0):
        """(factor values, [local level-grid nodes]) of the rank's patch preconditioner."""
        h = _vp()
        _check(lib().lorpc_dist_local_prec(self.h, int(local), ctypes.byref(h)))
        J, Lv = _ll(), _int()
        _check(lib().lorpc_prec_info(h, ctypes.byref(J), ctypes.byref(Lv)))
        fv, cn = _ll(), _ll()
        ln = (_ll * 8)()
        _check(lib().lorpc_prec_bytes(h, ctypes.byref(fv), ln, ctypes.byref(cn)))
        return fv.value, [ln[i] for i in range(Lv.value)]

    def apply(self, xs, ys):
        _check(lib().lorpc_dist_operator_apply(self.h, self._ptrs(xs), self._ptrs(ys)))

    def precond(self, rs, zs):
        _check(lib().lorpc_dist_precond_apply(self.h, self._ptrs(rs), self._ptrs(zs)))

    def pcg_solve(self, bs, xs, rtol, maxit=2000):
        rep, keep = _mkrep(maxit)
        _check(lib().lorpc_dist_pcg_solve(self.h, self._ptrs(bs), self._ptrs(xs), float(rtol), int(maxit),
                                          ctypes.byref(rep)))
        return _report(rep, maxit, keep)
