"""Python mirror of the reference's C++ API for the H² hot path, over the C ABI.

Names, argument meaning and error behaviour follow igabem
(/root/reference/proj/core/include/igabem): ``make_sphere`` / ``make_square``
(shapes.hpp), ``Pde`` (pde.hpp), ``Discretization`` (spaces.hpp),
``H2Options`` / ``AssemblyOptions`` (h2.hpp, assembly.hpp) and
``H2Matrix`` (h2.hpp:57-106).  Exceptions map the reference's C++ exception
types: std::invalid_argument -> ValueError, std::logic_error ->
LogicError, std::runtime_error -> RuntimeError, std::domain_error ->
DomainError.  There is no CPU fallback: every operator call runs the CUDA
kernels of libigabem_b200.so, and a missing library or device raises.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# IGB_B200_LIB: another build of the same library (A/B of compile-time variants)
_LIB_PATH = os.environ.get("IGB_B200_LIB") or os.path.join(_HERE, "libigabem_b200.so")
_LIB = None


class LogicError(RuntimeError):
    """std::logic_error"""


class DomainError(ValueError):
    """std::domain_error"""


class CudaError(RuntimeError):
    """device failure"""


_EXC = {1: ValueError, 2: LogicError, 3: RuntimeError, 4: DomainError, 5: CudaError}

LAPLACE, HELMHOLTZ, MAXWELL = 0, 1, 2
FAR, VERTEX, EDGE, COINCIDENT = 0, 1, 2, 3


class _DiscInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int) for n in ("dof_count", "element_count", "local_count", "level", "degree",
                                            "repetition", "kind", "patch_count")]


class _Opts(ctypes.Structure):
    _fields_ = [("m", ctypes.c_int), ("eta", ctypes.c_double), ("far_order", ctypes.c_int),
                ("sing_order", ctypes.c_int)]


class _Storage(ctypes.Structure):
    _fields_ = [("nearfield_entries", ctypes.c_size_t), ("farfield_entries", ctypes.c_size_t),
                ("total_bytes", ctypes.c_size_t)]


class _Times(ctypes.Structure):
    _fields_ = [(n, ctypes.c_double) for n in ("plan_host_ms", "upload_ms", "elements_ms", "images_ms",
                                               "couplings_ms", "regular_ms", "coincident_ms", "edge_ms",
                                               "vertex_ms", "device_total_ms", "wall_total_ms", "scatter_ms")]


class _SolverOpts(ctypes.Structure):
    _fields_ = [("tol", ctypes.c_double), ("max_iter", ctypes.c_int), ("restart", ctypes.c_int)]


class _SolveStats(ctypes.Structure):
    _fields_ = [("iterations", ctypes.c_int), ("residual", ctypes.c_double), ("converged", ctypes.c_int),
                ("seconds", ctypes.c_double)]


class _PatchDesc(ctypes.Structure):
    _fields_ = [("degree_u", ctypes.c_int), ("degree_v", ctypes.c_int), ("n_knots_u", ctypes.c_int),
                ("n_knots_v", ctypes.c_int), ("knots_u", ctypes.POINTER(ctypes.c_double)),
                ("knots_v", ctypes.POINTER(ctypes.c_double)), ("ctrl_w", ctypes.POINTER(ctypes.c_double)),
                ("weight", ctypes.POINTER(ctypes.c_double))]


SYMBOLS = (
    "igb_geometry_create", "igb_geometry_sphere", "igb_geometry_square", "igb_geometry_info",
    "igb_geometry_destroy", "igb_discretization_create", "igb_discretization_info", "igb_discretization_l2g",
    "igb_discretization_elements", "igb_classify_pair", "igb_discretization_destroy", "igb_h2_create", "igb_h2_create_ex", "igb_h2_create_dist", "igb_h2_dist_send_count",
    "igb_h2_dist_phase1", "igb_h2_dist_phase2",
    "igb_h2_dim", "igb_h2_apply", "igb_h2_apply_device", "igb_h2_storage_report", "igb_h2_counts",
    "igb_h2_near_pairs", "igb_h2_far_pairs", "igb_h2_tree", "igb_h2_near_blocks", "igb_h2_couplings",
    "igb_h2_moments", "igb_h2_images", "igb_h2_assembly_times", "igb_h2_device_bytes", "igb_h2_bench_apply",
    "igb_h2_gmres", "igb_h2_cg", "igb_rhs_points", "igb_rhs_assemble", "igb_potential", "igb_dense_assemble",
    "igb_h2_reassemble", "igb_h2_upload_bytes", "igb_h2_profile_apply", "igb_h2_bench_steps",
    "igb_h2_class_counts", "igb_h2_launch_counts", "igb_plan_create", "igb_plan_create_ex", "igb_plan_counts", "igb_plan_near_pairs",
    "igb_plan_far_pairs", "igb_plan_class_counts", "igb_plan_node_boxes", "igb_plan_partition", "igb_plan_owned", "igb_plan_singular_items",
    "igb_plan_destroy", "igb_h2_destroy", "igb_admissible", "igb_last_error", "igb_version",
    "igb_release_device_memory", "igb_h2_profile_kernels", "igb_h2_far_work", "igb_h2_leaf_blocks", "igb_h2_far_field", "igb_h2_dist_dof_mask",
)


def library_path() -> str:
    return _LIB_PATH


def lib():
    """Load libigabem_b200.so (built in-tree by __graft_entry__.build())."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
    L = ctypes.CDLL(_LIB_PATH)
    vp, i32, f64, i64, sz = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong, ctypes.c_size_t
    P = ctypes.POINTER
    L.igb_geometry_create.argtypes = [i32, P(_PatchDesc), P(vp)]
    L.igb_geometry_sphere.argtypes = [f64, P(f64), P(vp)]
    L.igb_geometry_square.argtypes = [P(vp)]
    L.igb_geometry_info.argtypes = [vp, P(i32), P(i32), P(i32)]
    L.igb_geometry_destroy.argtypes = [vp]
    L.igb_geometry_destroy.restype = None
    L.igb_discretization_create.argtypes = [vp, i32, f64, f64, i32, i32, i32, P(vp)]
    L.igb_discretization_info.argtypes = [vp, P(_DiscInfo)]
    L.igb_discretization_l2g.argtypes = [vp, P(i32), P(f64)]
    L.igb_discretization_elements.argtypes = [vp, P(i32), P(f64)]
    L.igb_classify_pair.argtypes = [vp, i32, i32, P(i32), P(i32)]
    L.igb_discretization_destroy.argtypes = [vp]
    L.igb_discretization_destroy.restype = None
    L.igb_h2_create.argtypes = [vp, P(_Opts), i32, P(vp)]
    L.igb_h2_create_ex.argtypes = [vp, P(_Opts), i32, i32, P(vp)]
    L.igb_h2_create_dist.argtypes = [vp, P(_Opts), i32, i32, i32, i32, P(vp)]
    L.igb_h2_dist_send_count.argtypes = [vp, P(sz)]
    L.igb_h2_dist_phase1.argtypes = [vp, vp, vp, vp]
    L.igb_h2_dist_phase2.argtypes = [vp, vp, vp, vp]
    L.igb_h2_dim.argtypes = [vp, P(i32)]
    L.igb_h2_apply.argtypes = [vp, P(f64), P(f64)]
    L.igb_h2_apply_device.argtypes = [vp, vp, vp, vp]
    L.igb_h2_storage_report.argtypes = [vp, P(_Storage)]
    L.igb_h2_counts.argtypes = [vp, P(i64), P(i64), P(i32)]
    L.igb_h2_near_pairs.argtypes = [vp, P(i32)]
    L.igb_h2_far_pairs.argtypes = [vp, P(i32)]
    L.igb_h2_tree.argtypes = [vp, P(i32), P(i32), P(i32), P(i32), P(f64)]
    L.igb_h2_near_blocks.argtypes = [vp, i64, i64, P(f64)]
    L.igb_h2_couplings.argtypes = [vp, i64, i64, P(f64)]
    L.igb_h2_moments.argtypes = [vp, P(f64)]
    L.igb_h2_images.argtypes = [vp, P(f64)]
    L.igb_h2_assembly_times.argtypes = [vp, P(_Times)]
    L.igb_h2_device_bytes.argtypes = [vp, P(sz), P(sz), P(sz)]
    L.igb_h2_bench_apply.argtypes = [vp, i32, P(ctypes.c_float), P(i32)]
    L.igb_h2_reassemble.argtypes = [vp, P(f64), P(i32)]
    L.igb_h2_upload_bytes.argtypes = [vp, P(sz)]
    L.igb_h2_profile_apply.argtypes = [vp, i32, P(f64)]
    L.igb_h2_class_counts.argtypes = [vp, P(i64)]
    L.igb_h2_launch_counts.argtypes = [vp, P(i32), P(i32)]
    L.igb_h2_bench_steps.argtypes = [vp, i32, i32, P(f64), P(f64)]
    L.igb_h2_destroy.argtypes = [vp]
    L.igb_h2_destroy.restype = None
    L.igb_plan_create.argtypes = [vp, P(_Opts), P(vp)]
    L.igb_plan_create_ex.argtypes = [vp, P(_Opts), i32, i32, P(vp)]
    L.igb_plan_counts.argtypes = [vp, P(i64), P(i64), P(i32)]
    L.igb_plan_near_pairs.argtypes = [vp, P(i32)]
    L.igb_plan_far_pairs.argtypes = [vp, P(i32)]
    L.igb_plan_class_counts.argtypes = [vp, P(i64)]
    L.igb_plan_node_boxes.argtypes = [vp, P(f64)]
    L.igb_plan_partition.argtypes = [vp, i32, i32, P(i32), P(i32), P(i32), P(i64), P(i64)]
    L.igb_plan_owned.argtypes = [vp, i32, i32, P(ctypes.c_ubyte), P(ctypes.c_ubyte)]
    L.igb_plan_singular_items.argtypes = [vp, i32, i32, P(ctypes.c_longlong), P(i32)]
    L.igb_plan_destroy.argtypes = [vp]
    L.igb_plan_destroy.restype = None
    L.igb_h2_gmres.argtypes = [vp, P(f64), P(f64), P(_SolverOpts), P(_SolveStats)]
    L.igb_h2_cg.argtypes = [vp, P(f64), P(f64), P(_SolverOpts), P(_SolveStats)]
    L.igb_rhs_points.argtypes = [vp, i32, i32, P(f64), P(i32)]
    L.igb_rhs_assemble.argtypes = [vp, i32, i32, P(f64), P(f64)]
    L.igb_potential.argtypes = [vp, P(f64), i32, P(f64), i32, i32, P(f64)]
    L.igb_dense_assemble.argtypes = [vp, i32, i32, i32, P(f64)]
    L.igb_admissible.argtypes = [P(f64), P(f64), f64]
    L.igb_last_error.argtypes = [ctypes.c_char_p, sz]
    L.igb_release_device_memory.argtypes = [i32]
    L.igb_h2_far_work.argtypes = [vp, P(i64)]
    L.igb_h2_leaf_blocks.argtypes = [vp, P(i64)]
    L.igb_h2_dist_dof_mask.argtypes = [vp, P(ctypes.c_ubyte)]
    L.igb_h2_far_field.argtypes = [vp, P(f64), P(f64), P(f64)]
    L.igb_h2_profile_kernels.argtypes = [vp, i32, i32, ctypes.c_char_p, P(f64), P(i32)]
    _LIB = L
    return L


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _check(rc):
    if rc != 0:
        buf = ctypes.create_string_buffer(1024)
        lib().igb_last_error(buf, 1024)
        raise _EXC.get(rc, RuntimeError)(buf.value.decode())


# ------------------------------------------------------------------ pde.hpp
@dataclass(frozen=True)
class Pde:
    """Pde{kind, kappa} (pde.hpp:9-27)."""
    kind: int = LAPLACE
    kappa: complex = 0j

    def is_complex(self):
        return self.kind != LAPLACE

    def is_vector(self):
        return self.kind == MAXWELL

    @staticmethod
    def laplace():
        return Pde(LAPLACE, 0j)

    @staticmethod
    def helmholtz(k):
        return Pde(HELMHOLTZ, complex(k))

    @staticmethod
    def maxwell(k):
        if complex(k) == 0:
            raise ValueError("Pde: Maxwell requires a nonzero wavenumber")
        return Pde(MAXWELL, complex(k))


# ------------------------------------------------------------- geometry.hpp
class Geometry:
    """Multi-patch NURBS geometry (geometry.hpp:38-76)."""

    def __init__(self, patches=None, _handle=None):
        if _handle is None:
            descs = (_PatchDesc * len(patches))()
            keep = []
            for i, p in enumerate(patches):
                ku = np.ascontiguousarray(p["knots_u"], dtype=np.float64)
                kv = np.ascontiguousarray(p["knots_v"], dtype=np.float64)
                cw = np.ascontiguousarray(p["ctrl_w"], dtype=np.float64)
                w = np.ascontiguousarray(p["weight"], dtype=np.float64)
                keep += [ku, kv, cw, w]
                descs[i] = _PatchDesc(p["degree_u"], p["degree_v"], len(ku), len(kv), _p(ku), _p(kv), _p(cw), _p(w))
            h = ctypes.c_void_p()
            _check(lib().igb_geometry_create(len(patches), descs, ctypes.byref(h)))
            _handle = h
        self._h = _handle
        n = [ctypes.c_int() for _ in range(3)]
        _check(lib().igb_geometry_info(self._h, *[ctypes.byref(x) for x in n]))
        self._np, self._ne, self._nv = (x.value for x in n)

    def patch_count(self):
        return self._np

    def edge_count(self):
        return self._ne

    def vertex_count(self):
        return self._nv

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.igb_geometry_destroy(self._h)
            self._h = None


def make_sphere(radius=1.0, center=(0.0, 0.0, 0.0)) -> Geometry:
    """Exact six-patch rational sphere (shapes.hpp:21-22, shapes.cpp:87-205)."""
    c = np.asarray(center, dtype=np.float64)
    h = ctypes.c_void_p()
    _check(lib().igb_geometry_sphere(float(radius), _p(c), ctypes.byref(h)))
    return Geometry(_handle=h)


def make_square() -> Geometry:
    """Unit square in z = 0 (shapes.hpp:16, shapes.cpp:28-30)."""
    h = ctypes.c_void_p()
    _check(lib().igb_geometry_square(ctypes.byref(h)))
    return Geometry(_handle=h)


# --------------------------------------------------------------- spaces.hpp
class Discretization:
    """Discrete ansatz space (spaces.hpp:37-105): Discretization(g, pde, degree, rep, level)."""

    def __init__(self, geometry: Geometry, pde: Pde, degree: int, rep: int, level: int):
        h = ctypes.c_void_p()
        _check(lib().igb_discretization_create(geometry._h, pde.kind, pde.kappa.real, pde.kappa.imag, int(degree),
                                               int(rep), int(level), ctypes.byref(h)))
        self._h = h
        self._geometry = geometry
        self._pde = pde
        info = _DiscInfo()
        _check(lib().igb_discretization_info(h, ctypes.byref(info)))
        self._info = info

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.igb_discretization_destroy(self._h)
            self._h = None

    def geometry(self):
        return self._geometry

    def pde(self):
        return self._pde

    def degree(self):
        return self._info.degree

    def repetition(self):
        return self._info.repetition

    def level(self):
        return self._info.level

    def dof_count(self):
        return self._info.dof_count

    def element_count(self):
        return self._info.element_count

    def local_count(self):
        return self._info.local_count

    def elements_per_patch(self):
        return 1 << (2 * self._info.level)

    def element_index(self, patch, ix, iy):
        return patch * self.elements_per_patch() + ix + (1 << self._info.level) * iy

    def local_to_global(self):
        n = self.element_count() * self.local_count()
        g = np.zeros(n, dtype=np.int32)
        s = np.zeros(n)
        _check(lib().igb_discretization_l2g(self._h, _p(g, ctypes.c_int), _p(s)))
        return g.reshape(self.element_count(), -1), s.reshape(self.element_count(), -1)

    def elements(self):
        ints = np.zeros((self.element_count(), 3), dtype=np.int32)
        dbl = np.zeros((self.element_count(), 9))
        _check(lib().igb_discretization_elements(self._h, _p(ints, ctypes.c_int), _p(dbl)))
        return ints, dbl

    def classify_pair(self, ea, eb):
        cls = ctypes.c_int()
        maps = np.zeros(6, dtype=np.int32)
        _check(lib().igb_classify_pair(self._h, int(ea), int(eb), ctypes.byref(cls), _p(maps, ctypes.c_int)))
        return cls.value, maps


# ------------------------------------------------------------------- h2.hpp
@dataclass
class AssemblyOptions:
    """AssemblyOptions (assembly.hpp:13-20); 0 -> P+2 (far) / P+3 (singular)."""
    far_order: int = 0
    sing_order: int = 0


@dataclass
class H2Options:
    """H2Options{m = 8, eta = 1.6, quad} (h2.hpp:11-15)."""
    m: int = 8
    eta: float = 1.6
    quad: AssemblyOptions = field(default_factory=AssemblyOptions)


@dataclass
class H2Storage:
    nearfield_entries: int
    farfield_entries: int
    total_bytes: int


def admissible(box_a, box_b, eta):
    """admissible() on boxes (min xyz, max xyz) (h2.cpp:92-97)."""
    a = np.ascontiguousarray(box_a, dtype=np.float64)
    b = np.ascontiguousarray(box_b, dtype=np.float64)
    return bool(lib().igb_admissible(_p(a), _p(b), float(eta)))


class H2Plan:
    """Block partition of H2Matrix (cluster tree, admissibility traversal, pair
    classification; h2.cpp:49-97,175-252).  device=None: all on the host;
    device=k: traversal, sort and transposes on CUDA device k (bit-identical)."""

    def __init__(self, disc: Discretization, opts: H2Options | None = None, device: int | None = None):
        opts = opts or H2Options()
        o = _Opts(int(opts.m), float(opts.eta), int(opts.quad.far_order), int(opts.quad.sing_order))
        h = ctypes.c_void_p()
        if device is None:
            _check(lib().igb_plan_create(disc._h, ctypes.byref(o), ctypes.byref(h)))
        else:
            _check(lib().igb_plan_create_ex(disc._h, ctypes.byref(o), 4, int(device), ctypes.byref(h)))
        self._h = h
        a, b, c = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int()
        _check(lib().igb_plan_counts(h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        self.near_count, self.far_count, self.node_count = a.value, b.value, c.value

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.igb_plan_destroy(self._h)
            self._h = None

    def nearfield_pairs(self):
        out = np.zeros((self.near_count, 2), dtype=np.int32)
        _check(lib().igb_plan_near_pairs(self._h, _p(out, ctypes.c_int)))
        return out

    def farfield_pairs(self):
        out = np.zeros((self.far_count, 2), dtype=np.int32)
        _check(lib().igb_plan_far_pairs(self._h, _p(out, ctypes.c_int)))
        return out

    def class_counts(self):
        out = np.zeros(4, dtype=np.int64)
        _check(lib().igb_plan_class_counts(self._h, _p(out, ctypes.c_longlong)))
        return dict(regular=int(out[0]), vertex=int(out[1]), edge=int(out[2]), coincident=int(out[3]))

    def node_boxes(self):
        """cluster boxes [node][min xyz, max xyz] (leaves: the element boxes)"""
        out = np.zeros((self.node_count, 6))
        _check(lib().igb_plan_node_boxes(self._h, _p(out, ctypes.c_double)))
        return out

    def partition(self, world, rank):
        c0, c1, ne = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        nn, nf = ctypes.c_longlong(), ctypes.c_longlong()
        _check(lib().igb_plan_partition(self._h, int(world), int(rank), ctypes.byref(c0), ctypes.byref(c1),
                                        ctypes.byref(ne), ctypes.byref(nn), ctypes.byref(nf)))
        return dict(clusters=(c0.value, c1.value), elements=ne.value, near=nn.value, far=nf.value)

    def owned(self, world, rank, n_elements):
        """(element mask, node mask) of one rank of the row-cluster partition"""
        em = np.zeros(n_elements, dtype=np.uint8)
        nm = np.zeros(self.node_count, dtype=np.uint8)
        _check(lib().igb_plan_owned(self._h, int(world), int(rank), _p(em, ctypes.c_ubyte), _p(nm, ctypes.c_ubyte)))
        return em.astype(bool), nm.astype(bool)

    def singular_items(self, world=1, rank=0):
        """(counts [regular, vertex, edge, coincident], equal): the singular items
        of one rank enumerated from the mesh topology alone, and whether they
        equal the near list's singular pairs (the device integrates the former
        before the block partition exists)."""
        counts = (ctypes.c_longlong * 4)()
        bad = ctypes.c_int()
        _check(lib().igb_plan_singular_items(self._h, int(world), int(rank), counts, ctypes.byref(bad)))
        return list(counts), bad.value == 0


class H2Matrix:
    """H2Matrix<Scalar>(disc, opts) (h2.hpp:57-106), assembled and applied on a B200.

    ``apply(x)`` takes and returns host numpy vectors (float64 for Laplace,
    complex128 for Helmholtz / Maxwell), like the reference's Eigen vectors."""

    def __init__(self, disc: Discretization, opts: H2Options | None = None, device: int = 0,
                 stored_couplings: bool | None = None, world: int = 1, rank: int = 0,
                 device_partition: Optional[bool] = None):
        opts = opts or H2Options()
        o = _Opts(int(opts.m), float(opts.eta), int(opts.quad.far_order), int(opts.quad.sing_order))
        h = ctypes.c_void_p()
        # stored_couplings: True -> stream stored couplings, False -> evaluate them
        # in every matvec, None -> chosen per kind and size (include/igabem_b200.h)
        # device_partition: None = the library's default (device), True / False force device / host
        flags = {True: 2, False: 8, None: 0}[stored_couplings] | {True: 4, False: 16, None: 0}[device_partition]
        if world == 1:
            _check(lib().igb_h2_create_ex(disc._h, ctypes.byref(o), int(device), flags, ctypes.byref(h)))
        else:
            _check(lib().igb_h2_create_dist(disc._h, ctypes.byref(o), int(device), flags, int(world), int(rank),
                                            ctypes.byref(h)))
        self.world, self.rank, self.device = world, rank, device
        self._h = h
        self._disc = disc
        self.opts = opts
        self.dtype = np.complex128 if disc.pde().is_complex() else np.float64
        n_near, n_far, n_nodes = ctypes.c_longlong(), ctypes.c_longlong(), ctypes.c_int()
        _check(lib().igb_h2_counts(h, ctypes.byref(n_near), ctypes.byref(n_far), ctypes.byref(n_nodes)))
        self.near_count, self.far_count, self.node_count = n_near.value, n_far.value, n_nodes.value
        self.nch = 4 if disc.pde().is_vector() else 1

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.igb_h2_destroy(self._h)
            self._h = None

    def rows(self):
        return self._disc.dof_count()

    cols = rows

    @property
    def stored_couplings(self):
        """whether this operator streams stored couplings (else evaluates them per matvec)"""
        return self.device_bytes()["far"] > 0

    def apply(self, x, out=None):
        """y = H x on host vectors; `out` (optional) receives y.  Page-locked
        buffers (e.g. torch pin_memory().numpy()) are transferred directly."""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        if x.shape != (self.rows(),):
            raise ValueError("H2Matrix::apply: dimension mismatch")
        if out is None:
            y = np.empty_like(x)
        else:
            y = out
            if y.shape != x.shape or y.dtype != x.dtype or not y.flags.c_contiguous:
                raise ValueError("H2Matrix::apply: out must be a contiguous vector like x")
        _check(lib().igb_h2_apply(self._h, _p(x.view(np.float64)), _p(y.view(np.float64))))
        return y

    __matmul__ = apply
    __mul__ = apply

    def apply_device(self, x_ptr: int, y_ptr: int, stream: int = 0):
        """Device-pointer matvec (x, y: CUDA device addresses of rows() scalars)."""
        _check(lib().igb_h2_apply_device(self._h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(y_ptr),
                                         ctypes.c_void_p(stream or None)))

    # multi-GPU phases (device pointers, cudaStream_t as int) -------------------
    def dist_send_count(self):
        n = ctypes.c_size_t()
        _check(lib().igb_h2_dist_send_count(self._h, ctypes.byref(n)))
        return n.value

    def dist_dof_mask(self):
        """bool per DOF: this rank's block rows contribute to y there"""
        m = np.zeros(self.rows(), dtype=np.uint8)
        _check(lib().igb_h2_dist_dof_mask(self._h, _p(m, ctypes.c_ubyte)))
        return m.astype(bool)

    def dist_phase1(self, x_ptr, send_ptr, stream=0):
        _check(lib().igb_h2_dist_phase1(self._h, ctypes.c_void_p(x_ptr), ctypes.c_void_p(send_ptr),
                                        ctypes.c_void_p(stream or None)))

    def dist_phase2(self, recv_ptr, y_ptr, stream=0):
        _check(lib().igb_h2_dist_phase2(self._h, ctypes.c_void_p(recv_ptr), ctypes.c_void_p(y_ptr),
                                        ctypes.c_void_p(stream or None)))

    def storage_report(self) -> H2Storage:
        s = _Storage()
        _check(lib().igb_h2_storage_report(self._h, ctypes.byref(s)))
        return H2Storage(s.nearfield_entries, s.farfield_entries, s.total_bytes)

    def nearfield_pairs(self):
        out = np.zeros((self.near_count, 2), dtype=np.int32)
        _check(lib().igb_h2_near_pairs(self._h, _p(out, ctypes.c_int)))
        return out

    def farfield_pairs(self):
        out = np.zeros((self.far_count, 2), dtype=np.int32)
        _check(lib().igb_h2_far_pairs(self._h, _p(out, ctypes.c_int)))
        return out

    def tree(self):
        n = self.node_count
        arrs = [np.zeros(n, dtype=np.int32) for _ in range(4)]
        boxes = np.zeros((n, 6))
        _check(lib().igb_h2_tree(self._h, *[_p(a, ctypes.c_int) for a in arrs], _p(boxes)))
        return dict(patch=arrs[0], level=arrs[1], sx=arrs[2], sy=arrs[3], box=boxes)

    # introspection ---------------------------------------------------------
    def near_blocks(self, first=0, count=None):
        count = self.near_count - first if count is None else count
        nl = self._disc.local_count()
        out = np.zeros((count, nl, nl), dtype=self.dtype)
        _check(lib().igb_h2_near_blocks(self._h, first, count, _p(out.view(np.float64))))
        return out

    def couplings(self, first=0, count=None):
        count = self.far_count - first if count is None else count
        mm = self.opts.m ** 2
        out = np.zeros((count, mm, mm), dtype=self.dtype)  # [q][mu][nu]
        _check(lib().igb_h2_couplings(self._h, first, count, _p(out.view(np.float64))))
        return np.ascontiguousarray(out.transpose(0, 2, 1))  # [q][nu][mu] = K(nu, mu)

    def moments(self):
        nl = self._disc.local_count()
        rows = self.nch * self.opts.m ** 2
        out = np.zeros((self._disc.element_count(), nl, rows))
        _check(lib().igb_h2_moments(self._h, _p(out)))
        return np.ascontiguousarray(out.transpose(0, 2, 1))  # [e][row][l]

    def images(self):
        out = np.zeros((self.node_count, self.opts.m ** 2, 3))
        _check(lib().igb_h2_images(self._h, _p(out)))
        return out

    def assembly_times(self):
        t = _Times()
        _check(lib().igb_h2_assembly_times(self._h, ctypes.byref(t)))
        return {n: getattr(t, n) for n, _ in _Times._fields_}

    def device_bytes(self):
        a, b, c = ctypes.c_size_t(), ctypes.c_size_t(), ctypes.c_size_t()
        _check(lib().igb_h2_device_bytes(self._h, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c)))
        return dict(near=a.value, far=b.value, moments=c.value)

    def reassemble(self):
        """Re-run the device assembly kernels (benchmark steps); returns (device ms, kernel launches)."""
        ms, n = ctypes.c_double(), ctypes.c_int()
        _check(lib().igb_h2_reassemble(self._h, ctypes.byref(ms), ctypes.byref(n)))
        return ms.value, n.value

    # profile_apply phases (serialised, CUDA events): near_rows = near-field
    # rows (overlapped with the far field in the graph), downward = downward
    # pass + leaf backward transform
    PHASES = ("coef", "leaf_up", "upward", "zero", "far", "near_rows", "downward", "scatter")

    def profile_apply(self, iters=10):
        """Per-phase matvec device time (ms, summed over iters)."""
        out = np.zeros(8)
        _check(lib().igb_h2_profile_apply(self._h, int(iters), _p(out)))
        return dict(zip(self.PHASES, out.tolist()))

    def profile_kernels(self, iters=10):
        """The matvec graph's own kernels, serialised, each timed with CUDA
        events: {role: ms summed over iters} (single-GPU level-split graph)."""
        names = ctypes.create_string_buffer(64 * 32)
        ms = np.zeros(64)
        n = ctypes.c_int()
        _check(lib().igb_h2_profile_kernels(self._h, int(iters), 64, names, _p(ms), ctypes.byref(n)))
        out = {}
        for k in range(n.value):
            key = names.raw[32 * k:32 * (k + 1)].split(b"\0")[0].decode()
            out[key] = out.get(key, 0.0) + float(ms[k])
        return out

    def far_field(self, x):
        """(up, down) after the far field of a matvec on x (phase 4 of apply,
        h2.cpp:312-326), each (node_count, nch * m^2): the far-field kernel's own
        output, for parity checks against the oracle."""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        if x.shape != (self.rows(),):
            raise ValueError("H2Matrix::far_field: dimension mismatch")
        shp = (self.node_count, self.nch * self.opts.m ** 2)
        up, down = np.zeros(shp, dtype=self.dtype), np.zeros(shp, dtype=self.dtype)
        _check(lib().igb_h2_far_field(self._h, _p(x.view(np.float64)), _p(up.view(np.float64)),
                                      _p(down.view(np.float64))))
        return up, down

    def far_sym_counts(self):
        """unordered far pairs evaluated per matvec by the symmetric far kernels:
        {'leaf': leaf level, 'coarse': above it}"""
        out = np.zeros(2, dtype=np.int64)
        _check(lib().igb_h2_far_work(self._h, _p(out, ctypes.c_longlong)))
        return dict(leaf=int(out[0]), coarse=int(out[1]))

    def leaf_blocks(self):
        """leaf-level far pairs applied as stored element blocks: (unordered pairs, bytes of
        their blocks, bytes of block rows -- near field + leaf blocks -- one matvec streams)"""
        out = np.zeros(3, dtype=np.int64)
        _check(lib().igb_h2_leaf_blocks(self._h, _p(out, ctypes.c_longlong)))
        return int(out[0]), int(out[1]), int(out[2])

    def bench_steps(self, steps, matvecs):
        """steps x (device assembly + matvecs matvecs): (total ms, assembly ms) from CUDA events."""
        t, a = ctypes.c_double(), ctypes.c_double()
        _check(lib().igb_h2_bench_steps(self._h, int(steps), int(matvecs), ctypes.byref(t), ctypes.byref(a)))
        return t.value, a.value

    def class_counts(self):
        """{'regular': ordered regular near pairs, 'vertex'/'edge'/'coincident': unique singular pairs}"""
        out = np.zeros(4, dtype=np.int64)
        _check(lib().igb_h2_class_counts(self._h, _p(out, ctypes.c_longlong)))
        return dict(regular=int(out[0]), vertex=int(out[1]), edge=int(out[2]), coincident=int(out[3]))

    def launch_counts(self):
        a, b = ctypes.c_int(), ctypes.c_int()
        _check(lib().igb_h2_launch_counts(self._h, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def upload_bytes(self):
        b = ctypes.c_size_t()
        _check(lib().igb_h2_upload_bytes(self._h, ctypes.byref(b)))
        return b.value

    def bench_apply(self, iters):
        ms = ctypes.c_float()
        launches = ctypes.c_int()
        _check(lib().igb_h2_bench_apply(self._h, int(iters), ctypes.byref(ms), ctypes.byref(launches)))
        return ms.value, launches.value


class DistH2Matrix:
    """Row-cluster-partitioned H2Matrix on one rank of a torch.distributed
    (NCCL) job: each rank assembles the block rows of its
    level-1 clusters; a matvec all-gathers the level>=1 up moments and
    all-reduces the partial result.  x and y are device tensors (replicated)."""

    def __init__(self, disc, opts=None, group=None, device=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        dev = torch.cuda.current_device() if device is None else device
        self.h = H2Matrix(disc, opts, device=dev, world=self.world, rank=self.rank)
        self.dtype = torch.complex128 if self.h.dtype == np.complex128 else torch.float64
        n = self.h.dist_send_count()
        dv = f"cuda:{dev}"
        self.send = torch.zeros(max(n, 1), dtype=self.dtype, device=dv)
        self.recv = torch.zeros(max(n, 1) * self.world, dtype=self.dtype, device=dv)
        self.n = n
        # y reduction over the cut DOFs only: masks of all ranks (once); a DOF
        # touched by several ranks is cut and summed by an all-reduce over the
        # compact cut list; every DOF is owned by the lowest rank touching it,
        # whose values all ranks all-gather to replicate y
        mine = torch.from_numpy(self.h.dist_dof_mask().astype(np.uint8))
        masks = [torch.zeros_like(mine) for _ in range(self.world)]
        self._gather_cpu_or_dev(masks, mine, dev)
        M = np.stack([m.numpy().astype(bool) for m in masks])
        touched = M.sum(axis=0)
        owner = np.argmax(M, axis=0)  # lowest touching rank (untouched DOFs: rank 0, value 0)
        self.cut = torch.from_numpy(np.flatnonzero(touched > 1)).to(dv)
        own = [np.flatnonzero(owner == r) for r in range(self.world)]
        self.own_max = max(len(o) for o in own)
        self.own_idx = [torch.from_numpy(o).to(dv) for o in own]
        self.cut_buf = torch.zeros(max(len(self.cut), 1), dtype=self.dtype, device=dv)
        self.own_buf = torch.zeros(self.own_max, dtype=self.dtype, device=dv)
        self.all_buf = torch.zeros(self.own_max * self.world, dtype=self.dtype, device=dv)
        oth = [(own[r], r * self.own_max + np.arange(len(own[r]))) for r in range(self.world) if r != self.rank]
        self.other_idx = torch.from_numpy(np.concatenate([o[0] for o in oth] or [np.zeros(0, np.int64)])).to(dv)
        self.other_pos = torch.from_numpy(np.concatenate([o[1] for o in oth] or [np.zeros(0, np.int64)])).to(dv)

    def rows(self):
        return self.h.rows()

    def apply(self, x, y=None):
        """y = H x with x, y replicated device tensors.  NCCL: the collectives run
        on the device tensors on torch's current stream; any other backend
        (gloo: CPU-only process groups, tests) stages them through host memory."""
        torch = self.torch
        y = torch.empty_like(x) if y is None else y
        stream = torch.cuda.current_stream().cuda_stream
        self.h.dist_phase1(x.data_ptr(), self.send.data_ptr(), stream)
        nccl = self.dist.get_backend(self.group) == "nccl"
        if nccl:
            self.dist.all_gather_into_tensor(self.recv, self.send, group=self.group)
        else:
            parts = [torch.empty(self.send.numel(), dtype=self.dtype) for _ in range(self.world)]
            self.dist.all_gather(parts, self.send.cpu(), group=self.group)
            self.recv.copy_(torch.cat(parts))
        self.h.dist_phase2(self.recv.data_ptr(), y.data_ptr(), torch.cuda.current_stream().cuda_stream)
        # cut DOFs: sum the partial values (fixed rank order in NCCL's / gloo's
        # reduction); then replicate y from the owners
        if len(self.cut):
            torch.index_select(y, 0, self.cut, out=self.cut_buf)
            self._allreduce(self.cut_buf)
            y.index_copy_(0, self.cut, self.cut_buf)
        mine = self.own_idx[self.rank]
        self.own_buf[:len(mine)] = y[mine]
        if nccl:
            self.dist.all_gather_into_tensor(self.all_buf, self.own_buf, group=self.group)
        else:
            parts = [torch.empty(self.own_max, dtype=self.dtype) for _ in range(self.world)]
            self.dist.all_gather(parts, self.own_buf.cpu(), group=self.group)
            self.all_buf.copy_(torch.cat(parts))
        y.index_copy_(0, self.other_idx, self.all_buf[self.other_pos])
        return y

    def _allreduce(self, t):
        if self.dist.get_backend(self.group) == "nccl":
            self.dist.all_reduce(t, group=self.group)
        else:
            h = t.cpu()
            self.dist.all_reduce(h, group=self.group)
            t.copy_(h)

    def _gather_cpu_or_dev(self, outs, t, dev):
        if self.dist.get_backend(self.group) == "nccl":
            o = [x.to(f"cuda:{dev}") for x in outs]
            self.dist.all_gather(o, t.to(f"cuda:{dev}"), group=self.group)
            for a, b in zip(outs, o):
                a.copy_(b.cpu())
        else:
            self.dist.all_gather(outs, t, group=self.group)


# ----------------------------------------------------------- SURVEY 8(f)
@dataclass
class SolverOptions:
    """SolverOptions{tol = 1e-8, max_iter = 1000, restart = 30} (solver.hpp:37-41)."""
    tol: float = 1e-8
    max_iter: int = 1000
    restart: int = 30


@dataclass
class SolveStats:
    iterations: int
    residual: float
    converged: bool
    seconds: float


def _solve(fn, h, b, opts):
    opts = opts or SolverOptions()
    b = np.ascontiguousarray(b, dtype=h.dtype)
    if b.shape != (h.rows(),):
        raise ValueError("solver: dimension mismatch")
    x = np.zeros_like(b)
    st = _SolveStats()
    o = _SolverOpts(float(opts.tol), int(opts.max_iter), int(opts.restart))
    _check(fn(h._h, _p(b.view(np.float64)), _p(x.view(np.float64)), ctypes.byref(o), ctypes.byref(st)))
    return x, SolveStats(st.iterations, st.residual, bool(st.converged), st.seconds)


def gmres(h: H2Matrix, b, opts: SolverOptions | None = None):
    """Restarted GMRES of solver.hpp:54-155 on the B200 operator; vectors stay in HBM."""
    return _solve(lib().igb_h2_gmres, h, b, opts)


def cg(h: H2Matrix, b, opts: SolverOptions | None = None):
    """CG of solver.hpp:159-200 on the B200 operator."""
    return _solve(lib().igb_h2_cg, h, b, opts)


def quadrature_points(disc: Discretization, quad_order=0, device=0):
    """Load-vector quadrature points, shape (elements, n^2, 3) (assembly.cpp:60-72)."""
    npe = ctypes.c_int()
    _check(lib().igb_rhs_points(disc._h, int(quad_order), int(device), None, ctypes.byref(npe)))
    out = np.zeros((disc.element_count(), npe.value, 3))
    _check(lib().igb_rhs_points(disc._h, int(quad_order), int(device), _p(out), ctypes.byref(npe)))
    return out


def compute_rhs(disc: Discretization, g, quad_order=0, device=0):
    """b_i = <g, phi_i> (compute_rhs / compute_rhs_complex / compute_rhs_maxwell,
    assembly.hpp:32-41).  g maps an (n, 3) array of points to n values
    (Maxwell: an (n, 3) array of complex field vectors)."""
    pts = quadrature_points(disc, quad_order, device)
    vals = np.asarray(g(pts.reshape(-1, 3)))
    pde = disc.pde()
    dt = np.complex128 if pde.is_complex() else np.float64
    if pde.is_vector():
        vals = np.ascontiguousarray(vals, dtype=np.complex128).reshape(-1, 3)
    else:
        vals = np.ascontiguousarray(vals, dtype=dt).reshape(-1)
    b = np.zeros(disc.dof_count(), dtype=dt)
    _check(lib().igb_rhs_assemble(disc._h, int(quad_order), int(device), _p(vals.view(np.float64)),
                                  _p(b.view(np.float64))))
    return b


def eval_potential(disc: Discretization, density, points, quad_order=10, device=0):
    """Single layer potential at points (operators.hpp:44-49); Maxwell: the
    electric field E = SL[j] + kappa^-2 grad SL[div j], shape (n, 3)."""
    pde = disc.pde()
    dt = np.complex128 if pde.is_complex() else np.float64
    dens = np.ascontiguousarray(density, dtype=dt)
    if dens.shape != (disc.dof_count(),):
        raise ValueError("eval_potential: density size does not match the space")
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    out = np.zeros((len(pts), 3) if pde.is_vector() else len(pts), dtype=dt)
    _check(lib().igb_potential(disc._h, _p(dens.view(np.float64)), len(pts), _p(pts), int(quad_order), int(device),
                               _p(out.view(np.float64))))
    return out


eval_maxwell_potential = eval_potential


def assemble_dense(disc: Discretization, opts: AssemblyOptions | None = None, device: int = 0):
    """assemble_dense / assemble_dense_complex (assembly.cpp:16-53) on the B200:
    the dense Galerkin matrix (dof_count x dof_count, float64 or complex128)."""
    opts = opts or AssemblyOptions()
    n = disc.dof_count()
    dt = np.complex128 if disc.pde().is_complex() else np.float64
    a = np.zeros((n, n), dtype=dt, order="F")
    _check(lib().igb_dense_assemble(disc._h, int(opts.far_order), int(opts.sing_order), int(device), _p(a)))
    return a


def make_sphere_grid(radius, n, center=(0.0, 0.0, 0.0)):
    """util.cpp:9-24: n x n points on a sphere (theta-major)."""
    if radius <= 0 or n < 1:
        raise ValueError("make_sphere_grid: bad arguments")
    k = np.arange(n)
    theta = np.pi * (k + 0.5) / n
    phi = 2.0 * np.pi * k / n
    th, ph = np.meshgrid(theta, phi, indexing="ij")
    pts = np.stack([np.sin(th) * np.cos(ph), np.sin(th) * np.sin(ph), np.cos(th)], axis=-1).reshape(-1, 3)
    return np.asarray(center, dtype=np.float64) + radius * pts
