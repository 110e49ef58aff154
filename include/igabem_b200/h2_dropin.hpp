// igabem_b200/h2_dropin.hpp -- header-only C++ drop-in for igabem::H2Matrix.
//
// For code written against the reference (igabem, proj/core/include/igabem/h2.hpp:57-106):
// replace `igabem::H2Matrix<Scalar> h(disc, opts);` by
// `igabem_b200::H2Matrix<Scalar> h(disc, opts);` -- same constructor arguments,
// same members (rows, cols, apply, operator*, storage_report, nearfield_pairs,
// farfield_pairs, tree), same exception types.  Assembly and matvec run on a
// B200 through the C ABI in ../igabem_b200.h; the Discretization is flattened
// through its public accessors (spaces.hpp:42-68, splines.hpp:53-67).  As with
// the reference (h2.hpp:95), the Discretization must outlive the H2Matrix:
// tree() returns an igabem::ClusterTree, which keeps a raw pointer to it
// (h2.cpp:49, 89); the device operator itself no longer reads it.
#pragma once

#include <igabem/h2.hpp>

#include <stdexcept>
#include <string>
#include <type_traits>
#include <utility>
#include <vector>

#include "../igabem_b200.h"

namespace igabem_b200 {

namespace detail {
inline void check(int rc) {
  if (rc == IGB_OK) return;
  char buf[1024];
  igb_last_error(buf, sizeof(buf));
  switch (rc) {
    case IGB_INVALID_ARGUMENT: throw std::invalid_argument(buf);
    case IGB_LOGIC_ERROR: throw std::logic_error(buf);
    case IGB_DOMAIN_ERROR: throw std::domain_error(buf);
    default: throw std::runtime_error(buf);
  }
}
}  // namespace detail

template <typename Scalar>
class H2Matrix {
  static_assert(std::is_same_v<Scalar, double> || std::is_same_v<Scalar, igabem::cplx>,
                "H2Matrix<Scalar>: double or std::complex<double>");

 public:
  using Vec = Eigen::Matrix<Scalar, Eigen::Dynamic, 1>;

  explicit H2Matrix(const igabem::Discretization& disc, igabem::H2Options opts = {}, int device = 0)
      : tree_(disc), dim_(disc.dof_count()) {
    if constexpr (std::is_same_v<Scalar, double>) {
      if (disc.pde().is_complex()) throw std::invalid_argument("H2Matrix<double>: complex kind");
    } else {
      if (!disc.pde().is_complex()) throw std::invalid_argument("H2Matrix<complex>: Laplace kind");
    }
    const auto& geo = disc.geometry();
    std::vector<igb_patch_desc> desc(geo.patch_count());
    std::vector<std::vector<double>> cw(geo.patch_count()), w(geo.patch_count());
    for (int p = 0; p < geo.patch_count(); ++p) {
      const igabem::PatchSurface& s = geo.patch(p);
      const int n = s.count_u() * s.count_v();
      cw[p].resize(3 * n);
      w[p].resize(n);
      for (int i = 0; i < n; ++i) {
        for (int c = 0; c < 3; ++c) cw[p][3 * i + c] = s.ctrl_w(c, i);
        w[p][i] = s.weight[i];
      }
      desc[p] = igb_patch_desc{s.kv_u.degree, s.kv_v.degree, static_cast<int>(s.kv_u.knots.size()),
                               static_cast<int>(s.kv_v.knots.size()), s.kv_u.knots.data(), s.kv_v.knots.data(),
                               cw[p].data(), w[p].data()};
    }
    igb_geometry* g = nullptr;
    detail::check(igb_geometry_create(geo.patch_count(), desc.data(), &g));
    igb_discretization* d = nullptr;
    const int kind = static_cast<int>(disc.pde().kind);
    const int rc = igb_discretization_create(g, kind, disc.pde().kappa.real(), disc.pde().kappa.imag(),
                                             disc.degree(), disc.repetition(), disc.level(), &d);
    igb_geometry_destroy(g);
    detail::check(rc);
    const igb_h2_opts o{opts.m, opts.eta, opts.quad.far_order, opts.quad.sing_order};
    const int rc2 = igb_h2_create(d, &o, device, &h_);
    igb_discretization_destroy(d);
    detail::check(rc2);
  }
  ~H2Matrix() {
    if (h_) igb_h2_destroy(h_);
  }
  H2Matrix(const H2Matrix&) = delete;
  H2Matrix& operator=(const H2Matrix&) = delete;
  H2Matrix(H2Matrix&& o) noexcept : tree_(std::move(o.tree_)), dim_(o.dim_), h_(std::exchange(o.h_, nullptr)) {}

  int rows() const { return dim_; }
  int cols() const { return dim_; }
  const igabem::ClusterTree& tree() const { return tree_; }

  Vec apply(const Vec& x) const {
    if (x.size() != dim_) throw std::invalid_argument("H2Matrix::apply: dimension mismatch");
    Vec y(dim_);
    detail::check(igb_h2_apply(h_, reinterpret_cast<const double*>(x.data()), reinterpret_cast<double*>(y.data())));
    return y;
  }
  Vec operator*(const Vec& x) const { return apply(x); }

  igabem::H2Storage storage_report() const {
    igb_h2_storage s{};
    detail::check(igb_h2_storage_report(h_, &s));
    igabem::H2Storage out;
    out.nearfield_entries = s.nearfield_entries;
    out.farfield_entries = s.farfield_entries;
    out.total_bytes = s.total_bytes;
    return out;
  }
  std::vector<std::pair<int, int>> nearfield_pairs() const { return pairs(true); }
  std::vector<std::pair<int, int>> farfield_pairs() const { return pairs(false); }

  igb_h2* handle() const { return h_; }

 private:
  std::vector<std::pair<int, int>> pairs(bool near) const {
    long long nn = 0, nf = 0;
    int nodes = 0;
    detail::check(igb_h2_counts(h_, &nn, &nf, &nodes));
    std::vector<int> buf(2 * (near ? nn : nf));
    detail::check(near ? igb_h2_near_pairs(h_, buf.data()) : igb_h2_far_pairs(h_, buf.data()));
    std::vector<std::pair<int, int>> out(buf.size() / 2);
    for (size_t i = 0; i < out.size(); ++i) out[i] = {buf[2 * i], buf[2 * i + 1]};
    return out;
  }

  igabem::ClusterTree tree_;
  int dim_;
  igb_h2* h_ = nullptr;
};

}  // namespace igabem_b200
