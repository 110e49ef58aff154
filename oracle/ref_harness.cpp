// ============================================================================
// oracle/ref_harness.cpp -- TEST INFRASTRUCTURE ONLY.
//
// extern "C" driver of the *reference itself* (igabem, compiled from
// /root/reference/proj/core/src against oracle/shim into oracle/_ref/): the
// checker that pins oracle/igb_oracle.cpp and produces tests/golden/, and the
// `kind: "reference"` CPU baseline of bench.py.  It only calls the reference's
// public API (Discretization, H2Matrix, assemble_dense, solvers, potentials)
// and its internal pair integration (src/pair_integration.hpp) for per-pair
// near-field blocks.
// ============================================================================
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "igabem/assembly.hpp"
#include "igabem/h2.hpp"
#include "igabem/operators.hpp"
#include "igabem/shapes.hpp"
#include "igabem/solver.hpp"
#include "pair_integration.hpp"

using namespace igabem;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = std::string("invalid_argument: ") + e.what();
    return 1;
  } catch (const std::logic_error& e) {
    g_err = std::string("logic_error: ") + e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = std::string("runtime_error: ") + e.what();
    return 3;
  }
}
struct RDisc {
  std::shared_ptr<const Geometry> geom;
  std::unique_ptr<Discretization> disc;
};
struct RH2 {
  RDisc* d;
  std::unique_ptr<H2Matrix<double>> real;
  std::unique_ptr<H2Matrix<cplx>> cx;
};
}  // namespace

extern "C" {

int ref_last_error(char* buf, int n) {
  std::snprintf(buf, n, "%s", g_err.c_str());
  return static_cast<int>(g_err.size());
}

int ref_gauss(int n, double* nodes, double* weights) {
  return guard([&] {
    const auto& r = gauss_rule(n);
    for (int i = 0; i < n; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
  });
}

int ref_pair_rule(int cls, int n, double* out, long long* count) {
  return guard([&] {
    const auto& r = pair_rule(static_cast<PairClass>(cls), n);
    *count = static_cast<long long>(r.size());
    if (out)
      for (size_t i = 0; i < r.size(); ++i) {
        out[5 * i] = r[i].ua;
        out[5 * i + 1] = r[i].va;
        out[5 * i + 2] = r[i].ub;
        out[5 * i + 3] = r[i].vb;
        out[5 * i + 4] = r[i].w;
      }
  });
}

// geom: 0 make_sphere(radius, center), 1 make_square(); kind 0/1/2
int ref_disc_create(int geom, double radius, const double* center, int kind, double kre, double kim, int P,
                    int rep, int L, void** out) {
  return guard([&] {
    auto d = std::make_unique<RDisc>();
    d->geom = std::make_shared<const Geometry>(
        geom == 0 ? make_sphere(radius, Eigen::Vector3d(center[0], center[1], center[2])) : make_square());
    Pde pde = kind == 0 ? Pde::laplace() : (kind == 1 ? Pde::helmholtz(cplx(kre, kim)) : Pde::maxwell(cplx(kre, kim)));
    d->disc = std::make_unique<Discretization>(d->geom, pde, P, rep, L);
    *out = d.release();
  });
}
void ref_disc_destroy(void* d) { delete static_cast<RDisc*>(d); }

void ref_disc_info(void* dp, int* out) {
  const Discretization& d = *static_cast<RDisc*>(dp)->disc;
  out[0] = d.dof_count();
  out[1] = d.element_count();
  out[2] = d.local_count();
  out[3] = d.geometry().patch_count();
  out[4] = d.level();
  out[5] = d.degree();
  out[6] = static_cast<int>(d.geometry().edge_idents().size());
  out[7] = static_cast<int>(d.geometry().vertex_idents().size());
}
void ref_disc_l2g(void* dp, int* l2g, double* sign) {
  const Discretization& d = *static_cast<RDisc*>(dp)->disc;
  for (int e = 0; e < d.element_count(); ++e)
    for (int l = 0; l < d.local_count(); ++l) {
      l2g[e * d.local_count() + l] = d.local_to_global(e, l);
      sign[e * d.local_count() + l] = d.local_sign(e, l);
    }
}
void ref_disc_elements(void* dp, int* ints, double* dbl) {
  const Discretization& d = *static_cast<RDisc*>(dp)->disc;
  for (int e = 0; e < d.element_count(); ++e) {
    const Element& el = d.element(e);
    ints[3 * e] = el.patch;
    ints[3 * e + 1] = el.ix;
    ints[3 * e + 2] = el.iy;
    double* o = dbl + 9 * e;
    o[0] = el.h;
    o[1] = el.origin.x();
    o[2] = el.origin.y();
    for (int k = 0; k < 3; ++k) {
      o[3 + k] = el.box.min()[k];
      o[6 + k] = el.box.max()[k];
    }
  }
}
void ref_patch(void* dp, int p, int* sizes, double* ku, double* kv, double* cw, double* w) {
  const PatchSurface& s = static_cast<RDisc*>(dp)->disc->geometry().patch(p);
  sizes[0] = s.kv_u.degree;
  sizes[1] = s.kv_v.degree;
  sizes[2] = static_cast<int>(s.kv_u.knots.size());
  sizes[3] = static_cast<int>(s.kv_v.knots.size());
  if (ku) std::copy(s.kv_u.knots.begin(), s.kv_u.knots.end(), ku);
  if (kv) std::copy(s.kv_v.knots.begin(), s.kv_v.knots.end(), kv);
  const int n = s.count_u() * s.count_v();
  if (cw)
    for (int i = 0; i < n; ++i)
      for (int c = 0; c < 3; ++c) cw[3 * i + c] = s.ctrl_w(c, i);
  if (w)
    for (int i = 0; i < n; ++i) w[i] = s.weight[i];
}
void ref_edges(void* dp, int* out) {
  int i = 0;
  for (const auto& e : static_cast<RDisc*>(dp)->disc->geometry().edge_idents()) {
    out[i++] = e.patch_a;
    out[i++] = e.edge_a;
    out[i++] = e.patch_b;
    out[i++] = e.edge_b;
    out[i++] = e.reversed ? 1 : 0;
  }
}
int ref_frame(void* dp, int p, double u, double v, double* out) {
  return guard([&] {
    const auto f = static_cast<RDisc*>(dp)->disc->geometry().frame(p, u, v);
    for (int k = 0; k < 3; ++k) {
      out[k] = f.x[k];
      out[3 + k] = f.du[k];
      out[6 + k] = f.dv[k];
      out[9 + k] = f.normal[k];
    }
    out[12] = f.sqrt_g;
  });
}
int ref_sample_shapes(void* dp, int e, double u, double v, double* value, double* field, double* div) {
  return guard([&] {
    const Discretization& d = *static_cast<RDisc*>(dp)->disc;
    const auto s = d.sample_shapes(e, u, v);
    for (int l = 0; l < d.local_count(); ++l) {
      if (value && s.value.size()) value[l] = s.value[l];
      if (field && s.field.size())
        for (int k = 0; k < 3; ++k) field[k * d.local_count() + l] = s.field(k, l);
      if (div && s.divergence.size()) div[l] = s.divergence[l];
    }
  });
}
int ref_classify(void* dp, int ea, int eb, int* maps) {
  const auto info = static_cast<RDisc*>(dp)->disc->classify_pair(ea, eb);
  if (maps) {
    maps[0] = info.map_a.swap; maps[1] = info.map_a.flip_u; maps[2] = info.map_a.flip_v;
    maps[3] = info.map_b.swap; maps[4] = info.map_b.flip_u; maps[5] = info.map_b.flip_v;
  }
  return static_cast<int>(info.cls);
}

// near-field blocks of a pair list via the reference's pair_block (the code
// H2Matrix::build_blocks runs per near pair, h2.cpp:236-243)
int ref_pair_blocks(void* dp, const int* pairs, long long npairs, int far_order, int sing_order, double* out) {
  return guard([&] {
    const Discretization& d = *static_cast<RDisc*>(dp)->disc;
    AssemblyOptions opts{far_order, sing_order};
    const int nl = d.local_count(), nfar = opts.resolved_far(d.degree()), nsing = opts.resolved_sing(d.degree());
    auto run = [&](auto tag) {
      using S = decltype(tag);
      std::vector<detail::FarCache<S>> caches(d.element_count());
      std::vector<char> need(d.element_count(), 0);
      for (long long q = 0; q < npairs; ++q) need[pairs[2 * q]] = need[pairs[2 * q + 1]] = 1;
#pragma omp parallel for schedule(dynamic, 16)
      for (int e = 0; e < d.element_count(); ++e)
        if (need[e]) caches[e] = detail::make_far_cache<S>(d, e, nfar);
#pragma omp parallel for schedule(dynamic, 1)
      for (long long q = 0; q < npairs; ++q) {
        const auto b = detail::pair_block<S>(d, caches, pairs[2 * q], pairs[2 * q + 1], nsing);
        std::memcpy(out + static_cast<size_t>(q) * nl * nl * (sizeof(S) / 8), b.data(), sizeof(S) * nl * nl);
      }
    };
    if (d.pde().is_complex()) run(cplx{}); else run(double{});
  });
}
int ref_dense(void* dp, int far_order, int sing_order, double* A) {
  return guard([&] {
    const Discretization& d = *static_cast<RDisc*>(dp)->disc;
    AssemblyOptions opts{far_order, sing_order};
    if (d.pde().is_complex()) {
      const auto a = assemble_dense_complex(d, opts);
      std::memcpy(A, a.data(), sizeof(cplx) * a.size());
    } else {
      const auto a = assemble_dense(d, opts);
      std::memcpy(A, a.data(), sizeof(double) * a.size());
    }
  });
}

int ref_h2_create(void* dp, int m, double eta, int far_order, int sing_order, int /*flags*/, void** out) {
  return guard([&] {
    auto h = std::make_unique<RH2>();
    h->d = static_cast<RDisc*>(dp);
    H2Options o;
    o.m = m;
    o.eta = eta;
    o.quad = AssemblyOptions{far_order, sing_order};
    if (h->d->disc->pde().is_complex())
      h->cx = std::make_unique<H2Matrix<cplx>>(*h->d->disc, o);
    else
      h->real = std::make_unique<H2Matrix<double>>(*h->d->disc, o);
    *out = h.release();
  });
}
void ref_h2_destroy(void* h) { delete static_cast<RH2*>(h); }

// out: near_count, far_count, node_count, near_entries, far_entries, total_bytes, nch, m
void ref_h2_info(void* hp, long long* out) {
  RH2* h = static_cast<RH2*>(hp);
  auto fill = [&](auto& H) {
    out[0] = static_cast<long long>(H.nearfield_pairs().size());
    out[1] = static_cast<long long>(H.farfield_pairs().size());
    out[2] = H.tree().node_count();
    const auto s = H.storage_report();
    out[3] = static_cast<long long>(s.nearfield_entries);
    out[4] = static_cast<long long>(s.farfield_entries);
    out[5] = static_cast<long long>(s.total_bytes);
    out[6] = h->d->disc->pde().is_vector() ? 4 : 1;
    out[7] = 0;
  };
  if (h->real) fill(*h->real); else fill(*h->cx);
}
void ref_h2_near_pairs(void* hp, int* out) {
  RH2* h = static_cast<RH2*>(hp);
  const auto p = h->real ? h->real->nearfield_pairs() : h->cx->nearfield_pairs();
  for (size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].first;
    out[2 * i + 1] = p[i].second;
  }
}
void ref_h2_far_pairs(void* hp, int* out) {
  RH2* h = static_cast<RH2*>(hp);
  const auto p = h->real ? h->real->farfield_pairs() : h->cx->farfield_pairs();
  for (size_t i = 0; i < p.size(); ++i) {
    out[2 * i] = p[i].first;
    out[2 * i + 1] = p[i].second;
  }
}
void ref_h2_boxes(void* hp, double* out) {
  RH2* h = static_cast<RH2*>(hp);
  const ClusterTree& t = h->real ? h->real->tree() : h->cx->tree();
  for (int i = 0; i < t.node_count(); ++i)
    for (int k = 0; k < 3; ++k) {
      out[6 * i + k] = t.node(i).box.min()[k];
      out[6 * i + 3 + k] = t.node(i).box.max()[k];
    }
}
int ref_h2_apply(void* hp, const double* x, double* y) {
  return guard([&] {
    RH2* h = static_cast<RH2*>(hp);
    const int n = h->d->disc->dof_count();
    if (h->real) {
      Eigen::VectorXd xv(n);
      std::memcpy(xv.data(), x, sizeof(double) * n);
      const Eigen::VectorXd yv = h->real->apply(xv);
      std::memcpy(y, yv.data(), sizeof(double) * n);
    } else {
      Eigen::VectorXcd xv(n);
      std::memcpy(xv.data(), x, sizeof(cplx) * n);
      const Eigen::VectorXcd yv = h->cx->apply(xv);
      std::memcpy(y, yv.data(), sizeof(cplx) * n);
    }
  });
}
// load vectors with the reference's compute_rhs* (assembly.cpp:108-133) for
// built-in data: 0 Laplace point source at q[0..2]; 1 Helmholtz point source
// (reference kernel e^{-i k r}/(4 pi r)); 2 Maxwell dipole at q[0..2] with
// moment q[3..5]; 3 Maxwell plane wave E = -pol e^{-i k d.x}, d = q[0..2],
// pol = q[3..5]; 4 outgoing e^{+i k r}/(4 pi r) point source
int ref_rhs(void* dp, int data, const double* q, int order, double* out) {
  return guard([&] {
    const Discretization& d = *static_cast<RDisc*>(dp)->disc;
    const Eigen::Vector3d a(q[0], q[1], q[2]), bq(q[3], q[4], q[5]);
    const cplx kap = d.pde().kappa;
    if (data == 0) {
      const auto b = compute_rhs(d, [&](const Eigen::Vector3d& x) { return laplace_point_source(x, a); }, order);
      std::memcpy(out, b.data(), sizeof(double) * b.size());
    } else if (data == 1 || data == 4) {
      const auto b = compute_rhs_complex(
          d,
          [&](const Eigen::Vector3d& x) {
            const cplx v = helmholtz_point_source(x, a, kap);
            return data == 1 ? v : std::conj(v);
          },
          order);
      std::memcpy(out, b.data(), sizeof(cplx) * b.size());
    } else {
      const auto b = compute_rhs_maxwell(
          d,
          [&](const Eigen::Vector3d& x) -> Eigen::Vector3cd {
            if (data == 2) return maxwell_dipole(x, a, bq, kap);
            const cplx ph = std::exp(cplx(0, -1) * kap * a.dot(x));
            return -(ph * bq.cast<cplx>());
          },
          order);
      std::memcpy(out, b.data(), sizeof(cplx) * b.size());
    }
  });
}
// gmres (method 0) or cg (1) of solver.hpp on the reference H2Matrix
int ref_solve(void* hp, int method, const double* b, double tol, int max_iter, int restart, double* x,
              double* stats) {
  return guard([&] {
    RH2* h = static_cast<RH2*>(hp);
    const int n = h->d->disc->dof_count();
    SolverOptions o{tol, max_iter, restart};
    auto run = [&](auto& H, auto tag) {
      using S = decltype(tag);
      using Vec = Eigen::Matrix<S, Eigen::Dynamic, 1>;
      Vec bv(n);
      std::memcpy(bv.data(), b, sizeof(S) * n);
      LinearOperator<S> op{n, [&H](const Vec& v) { return H.apply(v); }};
      auto [xv, st] = method == 0 ? gmres(op, bv, o) : cg(op, bv, o);
      std::memcpy(x, xv.data(), sizeof(S) * n);
      stats[0] = st.iterations;
      stats[1] = st.residual;
      stats[2] = st.converged ? 1 : 0;
      stats[3] = st.seconds;
    };
    if (h->real) run(*h->real, double{}); else run(*h->cx, cplx{});
  });
}
// eval_potential / eval_maxwell_potential (operators.cpp:112-208)
int ref_potential(void* dp, const double* dens, int npts, const double* pts, int order, double* out) {
  return guard([&] {
    const Discretization& d = *static_cast<RDisc*>(dp)->disc;
    std::vector<Eigen::Vector3d> p(npts);
    for (int i = 0; i < npts; ++i) p[i] = Eigen::Vector3d(pts[3 * i], pts[3 * i + 1], pts[3 * i + 2]);
    const int n = d.dof_count();
    if (!d.pde().is_complex()) {
      Eigen::VectorXd rho(n);
      std::memcpy(rho.data(), dens, sizeof(double) * n);
      const auto u = eval_potential(d, rho, p, order);
      std::memcpy(out, u.data(), sizeof(double) * npts);
    } else {
      Eigen::VectorXcd rho(n);
      std::memcpy(rho.data(), dens, sizeof(cplx) * n);
      if (d.pde().is_vector()) {
        const auto e = eval_maxwell_potential(d, rho, p, order);
        for (int i = 0; i < npts; ++i)
          for (int k = 0; k < 3; ++k) reinterpret_cast<cplx*>(out)[3 * i + k] = e(k, i);
      } else {
        const auto u = eval_potential(d, rho, p, order);
        std::memcpy(out, u.data(), sizeof(cplx) * npts);
      }
    }
  });
}

int ref_admissible(const double* boxa, const double* boxb, double eta) {
  ClusterNode a{0, 0, 0, 0, {}}, b{0, 0, 0, 0, {}};
  a.box = Eigen::AlignedBox3d(Eigen::Vector3d(boxa[0], boxa[1], boxa[2]), Eigen::Vector3d(boxa[3], boxa[4], boxa[5]));
  b.box = Eigen::AlignedBox3d(Eigen::Vector3d(boxb[0], boxb[1], boxb[2]), Eigen::Vector3d(boxb[3], boxb[4], boxb[5]));
  return admissible(a, b, eta) ? 1 : 0;
}

}  // extern "C"
