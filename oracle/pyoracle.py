"""ctypes binding of oracle/liborc.so -- TEST INFRASTRUCTURE ONLY.

The CPU restatement of the reference (igabem, /root/reference/proj/core) used
as the parity checker by tests/, __graft_entry__.smoke() and bench.py's CPU
baseline leg.  The product package never imports this module.
"""
import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

KIND = {"laplace": 0, "helmholtz": 1, "maxwell": 2}
FAR, VERTEX, EDGE, COINCIDENT = 0, 1, 2, 3


class _Prefixed:
    """exposes the `ref_*` symbols of oracle/_ref/libigabem_ref.so under the `orc_*` names"""

    def __init__(self, cdll, prefix):
        self._cdll, self._prefix = cdll, prefix

    def __getattr__(self, name):
        f = getattr(self._cdll, self._prefix + name[len("orc_"):])
        setattr(self, name, f)
        return f


def _sig(L, name, argtypes, optional=False):
    try:
        getattr(L, name).argtypes = argtypes
    except AttributeError:
        if PREFIX == "orc_" and not optional:
            raise  # the restatement must export the path; the reference harness a subset


LIB_PATH = os.path.join(_HERE, "liborc.so")
PREFIX = "orc_"


def lib():
    global _LIB
    if _LIB is None:
        path = LIB_PATH
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run __graft_entry__.build()")
        L = ctypes.CDLL(path)
        if PREFIX != "orc_":
            L = _Prefixed(L, PREFIX)
        vp, i32, f64, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_double, ctypes.c_longlong
        P = ctypes.POINTER
        _sig(L, "orc_disc_create", [i32, f64, P(f64), i32, f64, f64, i32, i32, i32, P(vp)])
        _sig(L, "orc_disc_destroy", [vp])
        _sig(L, "orc_disc_info", [vp, P(i32)])
        _sig(L, "orc_disc_l2g", [vp, P(i32), P(f64)])
        _sig(L, "orc_disc_elements", [vp, P(i32), P(f64)])
        _sig(L, "orc_patch", [vp, i32, P(i32), P(f64), P(f64), P(f64), P(f64)])
        _sig(L, "orc_edges", [vp, P(i32)])
        _sig(L, "orc_frame", [vp, i32, f64, f64, P(f64)])
        _sig(L, "orc_sample_shapes", [vp, i32, f64, f64, P(f64), P(f64), P(f64)])
        _sig(L, "orc_classify", [vp, i32, i32, P(i32)])
        _sig(L, "orc_pair_blocks", [vp, P(i32), i64, i32, i32, P(f64)])
        _sig(L, "orc_dense", [vp, i32, i32, P(f64)])
        _sig(L, "orc_h2_create", [vp, i32, f64, i32, i32, i32, P(vp)])
        _sig(L, "orc_h2_destroy", [vp])
        _sig(L, "orc_h2_info", [vp, P(i64)])
        _sig(L, "orc_h2_near_pairs", [vp, P(i32)])
        _sig(L, "orc_h2_far_pairs", [vp, P(i32)])
        _sig(L, "orc_h2_near_blocks", [vp, i64, i64, P(f64)])
        _sig(L, "orc_h2_couplings", [vp, i64, i64, P(f64)])
        _sig(L, "orc_h2_moments", [vp, P(f64)])
        _sig(L, "orc_h2_images", [vp, P(f64)])
        _sig(L, "orc_h2_boxes", [vp, P(f64)])
        _sig(L, "orc_h2_transfer", [vp, P(f64), P(f64)])
        _sig(L, "orc_h2_apply", [vp, P(f64), P(f64)])
        _sig(L, "orc_gauss", [i32, P(f64), P(f64)])
        _sig(L, "orc_pair_rule", [i32, i32, P(f64), P(i64)])
        _sig(L, "orc_admissible", [P(f64), P(f64), f64])
        # 8(f) pipeline: exported by the reference harness (oracle/_ref) only
        _sig(L, "orc_h2_apply_ex", [vp, P(f64), P(f64), P(f64), P(f64), P(f64)], optional=True)
        _sig(L, "orc_h2_probe", [vp, P(f64), P(f64), i32, P(i32), P(f64), i32, P(i32), P(f64)], optional=True)
        _sig(L, "orc_rhs", [vp, i32, P(f64), i32, P(f64)], optional=True)
        _sig(L, "orc_solve", [vp, i32, P(f64), f64, i32, i32, P(f64), P(f64)], optional=True)
        _sig(L, "orc_potential", [vp, P(f64), i32, P(f64), i32, P(f64)], optional=True)
        _sig(L, "orc_last_error", [ctypes.c_char_p, i32])
        _LIB = L
    return _LIB


def _p(a, t=ctypes.c_double):
    return a.ctypes.data_as(ctypes.POINTER(t))


def _check(rc):
    if rc != 0:
        buf = ctypes.create_string_buffer(512)
        lib().orc_last_error(buf, 512)
        msg = buf.value.decode()
        exc = {1: ValueError, 2: RuntimeError}.get(rc, RuntimeError)
        raise exc(msg)


def gauss(n):
    x = np.zeros(n)
    w = np.zeros(n)
    _check(lib().orc_gauss(n, _p(x), _p(w)))
    return x, w


def pair_rule(cls, n):
    cnt = ctypes.c_longlong(0)
    _check(lib().orc_pair_rule(cls, n, None, ctypes.byref(cnt)))
    out = np.zeros((cnt.value, 5))
    _check(lib().orc_pair_rule(cls, n, _p(out), ctypes.byref(cnt)))
    return out


def admissible(boxa, boxb, eta):
    a = np.ascontiguousarray(boxa, dtype=np.float64)
    b = np.ascontiguousarray(boxb, dtype=np.float64)
    return bool(lib().orc_admissible(_p(a), _p(b), eta))


class Discretization:
    """Oracle twin of igabem::Discretization (spaces.hpp:37-105)."""

    def __init__(self, kind="laplace", degree=1, rep=1, level=1, kappa=0j, geometry="sphere",
                 radius=1.0, center=(0.0, 0.0, 0.0)):
        self.kind = kind
        self.kappa = complex(kappa)
        c = np.asarray(center, dtype=np.float64)
        h = ctypes.c_void_p()
        _check(lib().orc_disc_create(0 if geometry == "sphere" else 1, radius, _p(c), KIND[kind],
                                     self.kappa.real, self.kappa.imag, degree, rep, level, ctypes.byref(h)))
        self._h = h
        info = np.zeros(8, dtype=np.int32)
        lib().orc_disc_info(h, _p(info, ctypes.c_int))
        (self.dof_count, self.element_count, self.local_count, self.patch_count, self.level,
         self.degree, self.n_edges, self.n_vertices) = (int(v) for v in info)
        self.is_complex = kind != "laplace"
        self.dtype = np.complex128 if self.is_complex else np.float64

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.orc_disc_destroy(self._h)
            self._h = None

    def l2g(self):
        n = self.element_count * self.local_count
        g = np.zeros(n, dtype=np.int32)
        s = np.zeros(n)
        lib().orc_disc_l2g(self._h, _p(g, ctypes.c_int), _p(s))
        return g.reshape(self.element_count, -1), s.reshape(self.element_count, -1)

    def elements(self):
        ints = np.zeros((self.element_count, 3), dtype=np.int32)
        dbl = np.zeros((self.element_count, 9))
        lib().orc_disc_elements(self._h, _p(ints, ctypes.c_int), _p(dbl))
        return ints, dbl

    def patch(self, p):
        sz = np.zeros(4, dtype=np.int32)
        lib().orc_patch(self._h, p, _p(sz, ctypes.c_int), None, None, None, None)
        ku = np.zeros(sz[2])
        kv = np.zeros(sz[3])
        n = (sz[2] - sz[0] - 1) * (sz[3] - sz[1] - 1)
        cw = np.zeros((n, 3))
        w = np.zeros(n)
        lib().orc_patch(self._h, p, _p(sz, ctypes.c_int), _p(ku), _p(kv), _p(cw), _p(w))
        return dict(pu=int(sz[0]), pv=int(sz[1]), ku=ku, kv=kv, cw=cw, w=w)

    def edges(self):
        out = np.zeros((self.n_edges, 5), dtype=np.int32)
        lib().orc_edges(self._h, _p(out, ctypes.c_int))
        return out

    def frame(self, patch, u, v):
        out = np.zeros(13)
        _check(lib().orc_frame(self._h, patch, u, v, _p(out)))
        return dict(x=out[0:3], du=out[3:6], dv=out[6:9], normal=out[9:12], sqrt_g=out[12])

    def sample_shapes(self, e, u, v):
        nl = self.local_count
        if self.kind == "maxwell":
            f = np.zeros((3, nl))
            d = np.zeros(nl)
            _check(lib().orc_sample_shapes(self._h, e, u, v, None, _p(f), _p(d)))
            return dict(field=f, divergence=d)
        val = np.zeros(nl)
        _check(lib().orc_sample_shapes(self._h, e, u, v, _p(val), None, None))
        return dict(value=val)

    def classify_pair(self, ea, eb):
        maps = np.zeros(6, dtype=np.int32)
        cls = lib().orc_classify(self._h, ea, eb, _p(maps, ctypes.c_int))
        return cls, maps

    def pair_blocks(self, pairs, far_order=0, sing_order=0):
        pairs = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1, 2)
        nl = self.local_count
        out = np.zeros((len(pairs), nl, nl), dtype=self.dtype)
        _check(lib().orc_pair_blocks(self._h, _p(pairs, ctypes.c_int), len(pairs), far_order, sing_order,
                                     _p(out.view(np.float64))))
        # stored column-major per block: transpose to [la, lb]
        return np.ascontiguousarray(out.transpose(0, 2, 1))

    def rhs(self, data, params, order=0):
        """reference compute_rhs* for built-in data (see oracle/ref_harness.cpp ref_rhs)"""
        q = np.zeros(6)
        q[:len(params)] = params
        b = np.zeros(self.dof_count, dtype=self.dtype)
        _check(lib().orc_rhs(self._h, int(data), _p(q), int(order), _p(b.view(np.float64))))
        return b

    def potential(self, density, pts, order=10):
        dens = np.ascontiguousarray(density, dtype=self.dtype)
        pts = np.ascontiguousarray(pts, dtype=np.float64).reshape(-1, 3)
        out = np.zeros((len(pts), 3) if self.kind == "maxwell" else len(pts), dtype=self.dtype)
        _check(lib().orc_potential(self._h, _p(dens.view(np.float64)), len(pts), _p(pts), int(order),
                                   _p(out.view(np.float64))))
        return out

    def assemble_dense(self, far_order=0, sing_order=0):
        nd = self.dof_count
        a = np.zeros((nd, nd), dtype=self.dtype)
        _check(lib().orc_dense(self._h, far_order, sing_order, _p(a.view(np.float64))))
        return np.ascontiguousarray(a.T)  # column-major -> row-major


class H2Matrix:
    """Oracle twin of igabem::H2Matrix<Scalar> (h2.hpp:57-106).

    flags bit0 skips near-field quadrature (zero blocks), bit1 skips coupling
    sampling; used only to time the matvec on a bounded CPU budget."""

    def __init__(self, disc, m=8, eta=1.6, far_order=0, sing_order=0, flags=0):
        self.disc = disc
        h = ctypes.c_void_p()
        _check(lib().orc_h2_create(disc._h, m, eta, far_order, sing_order, flags, ctypes.byref(h)))
        self._h = h
        info = np.zeros(8, dtype=np.int64)
        lib().orc_h2_info(h, _p(info, ctypes.c_longlong))
        (self.near_count, self.far_count, self.node_count, self.nearfield_entries, self.farfield_entries,
         self.total_bytes, self.nch, self.m) = (int(v) for v in info)
        self.dtype = disc.dtype

    def __del__(self):
        if getattr(self, "_h", None) and _LIB is not None:
            _LIB.orc_h2_destroy(self._h)
            self._h = None

    def apply(self, x):
        x = np.ascontiguousarray(x, dtype=self.dtype)
        if x.shape != (self.disc.dof_count,):
            raise ValueError("H2Matrix::apply: dimension mismatch")
        y = np.zeros_like(x)
        _check(lib().orc_h2_apply(self._h, _p(x.view(np.float64)), _p(y.view(np.float64))))
        return y

    __matmul__ = apply

    def apply_ex(self, x):
        """(y, up, down after the far field (phase 4), down after the downward
        pass (phase 5)); up / down: (node_count, nch * m^2) (oracle only)"""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        y = np.zeros_like(x)
        shp = (self.node_count, self.nch * self.m * self.m)
        up, d4, d5 = (np.zeros(shp, dtype=self.dtype) for _ in range(3))
        _check(lib().orc_h2_apply_ex(self._h, _p(x.view(np.float64)), _p(y.view(np.float64)),
                                     _p(up.view(np.float64)), _p(d4.view(np.float64)), _p(d5.view(np.float64))))
        return y, up, d4, d5

    def probe(self, x, nodes=(), dofs=()):
        """(up of all nodes, phase-4 down of `nodes`, y at `dofs`) with apply()'s
        arithmetic, evaluating only what they depend on (oracle only; with
        flags bits 2/3 couplings / near blocks are computed where used)"""
        x = np.ascontiguousarray(x, dtype=self.dtype)
        nodes = np.ascontiguousarray(nodes, dtype=np.int32)
        dofs = np.ascontiguousarray(dofs, dtype=np.int32)
        ncol = self.nch * self.m * self.m
        up = np.zeros((self.node_count, ncol), dtype=self.dtype)
        d4 = np.zeros((max(len(nodes), 1), ncol), dtype=self.dtype)
        y = np.zeros(max(len(dofs), 1), dtype=self.dtype)
        _check(lib().orc_h2_probe(self._h, _p(x.view(np.float64)), _p(up.view(np.float64)), len(nodes),
                                  _p(nodes, ctypes.c_int), _p(d4.view(np.float64)), len(dofs), _p(dofs, ctypes.c_int),
                                  _p(y.view(np.float64))))
        return up, d4[:len(nodes)], y[:len(dofs)]

    def solve(self, b, method="gmres", tol=1e-8, max_iter=1000, restart=30):
        """reference gmres / cg (solver.hpp) on this H2Matrix"""
        b = np.ascontiguousarray(b, dtype=self.dtype)
        x = np.zeros_like(b)
        st = np.zeros(4)
        _check(lib().orc_solve(self._h, 0 if method == "gmres" else 1, _p(b.view(np.float64)), float(tol),
                               int(max_iter), int(restart), _p(x.view(np.float64)), _p(st)))
        return x, dict(iterations=int(st[0]), residual=float(st[1]), converged=bool(st[2]), seconds=float(st[3]))

    def nearfield_pairs(self):
        out = np.zeros((self.near_count, 2), dtype=np.int32)
        lib().orc_h2_near_pairs(self._h, _p(out, ctypes.c_int))
        return out

    def farfield_pairs(self):
        out = np.zeros((self.far_count, 2), dtype=np.int32)
        lib().orc_h2_far_pairs(self._h, _p(out, ctypes.c_int))
        return out

    def near_blocks(self, first=0, count=None):
        count = self.near_count - first if count is None else count
        nl = self.disc.local_count
        out = np.zeros((count, nl, nl), dtype=self.dtype)
        lib().orc_h2_near_blocks(self._h, first, count, _p(out.view(np.float64)))
        return np.ascontiguousarray(out.transpose(0, 2, 1))

    def couplings(self, first=0, count=None):
        count = self.far_count - first if count is None else count
        mm = self.m * self.m
        out = np.zeros((count, mm, mm), dtype=self.dtype)
        lib().orc_h2_couplings(self._h, first, count, _p(out.view(np.float64)))
        return np.ascontiguousarray(out.transpose(0, 2, 1))

    def moments(self):
        rows = self.nch * self.m * self.m
        nl = self.disc.local_count
        out = np.zeros((self.disc.element_count, nl, rows), dtype=self.dtype)
        lib().orc_h2_moments(self._h, _p(out.view(np.float64)))
        return np.ascontiguousarray(out.transpose(0, 2, 1))

    def images(self):
        out = np.zeros((self.node_count, self.m * self.m, 3))
        lib().orc_h2_images(self._h, _p(out))
        return out

    def boxes(self):
        out = np.zeros((self.node_count, 6))
        lib().orc_h2_boxes(self._h, _p(out))
        return out

    def transfer(self):
        tl = np.zeros((self.m, self.m), dtype=self.dtype)
        tr = np.zeros((self.m, self.m), dtype=self.dtype)
        lib().orc_h2_transfer(self._h, _p(tl.view(np.float64)), _p(tr.view(np.float64)))
        return tl.T.copy(), tr.T.copy()
