// Host setup for the B200 H² operator: geometry, discrete space, block
// partition.  See igb_host.hpp.  References are to /root/reference/proj/core.
#include "igb_host.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <omp.h>

#include <parallel/algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

namespace igb {

// ------------------------------------------------------------------ Box
void Box::set_empty() {
  for (int k = 0; k < 3; ++k) {
    mn[k] = std::numeric_limits<double>::max();
    mx[k] = std::numeric_limits<double>::lowest();
  }
}
void Box::extend(const V3& p) {
  for (int k = 0; k < 3; ++k) {
    mn[k] = std::min(mn[k], p[k]);
    mx[k] = std::max(mx[k], p[k]);
  }
}
void Box::extend(const Box& b) {
  for (int k = 0; k < 3; ++k) {
    mn[k] = std::min(mn[k], b.mn[k]);
    mx[k] = std::max(mx[k], b.mx[k]);
  }
}
double Box::diag_norm() const {
  return norm(V3(mx[0] - mn[0], mx[1] - mn[1], mx[2] - mn[2]));
}
double Box::exterior_distance(const Box& b) const {
  double d2 = 0;
  for (int k = 0; k < 3; ++k) {
    if (mn[k] > b.mx[k]) {
      const double aux = mn[k] - b.mx[k];
      d2 += aux * aux;
    } else if (b.mn[k] > mx[k]) {
      const double aux = b.mn[k] - mx[k];
      d2 += aux * aux;
    }
  }
  return std::sqrt(d2);
}

// -------------------------------------------------------------- splines
int KnotVector::find_span(double x) const {  // splines.cpp:20-38
  const int p = degree, k = size();
  if (x >= knots[k]) {
    int j = k - 1;
    while (knots[j + 1] <= knots[j]) --j;
    return j;
  }
  int lo = p, hi = k;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (x < knots[mid])
      hi = mid;
    else
      lo = mid;
  }
  return lo;
}
KnotVector make_knots(std::vector<double> k, int p) {  // splines.cpp:7-18
  if (p < 0) throw std::invalid_argument("KnotVector: negative degree");
  const int n = static_cast<int>(k.size());
  if (n - p - 1 <= p) throw std::invalid_argument("KnotVector: too few knots");
  for (int i = 0; i + 1 < n; ++i)
    if (k[i] > k[i + 1]) throw std::invalid_argument("KnotVector: knots not nondecreasing");
  for (int i = 0; i <= p; ++i)
    if (k[i] != k.front() || k[n - 1 - i] != k.back())
      throw std::invalid_argument("KnotVector: not clamped");
  KnotVector kv;
  kv.knots = std::move(k);
  kv.degree = p;
  return kv;
}
KnotVector make_uniform_knots(int p, int level, int rep) {  // splines.cpp:40-52
  if (p < 0 || level < 0) throw std::invalid_argument("make_uniform_knots: bad p/L");
  if (rep < 1 || rep > p + 1)
    throw std::invalid_argument("make_uniform_knots: knot repetition must be in [1, p+1]");
  const int nel = 1 << level;
  std::vector<double> k;
  for (int i = 0; i <= p; ++i) k.push_back(0.0);
  for (int i = 1; i < nel; ++i)
    for (int r = 0; r < rep; ++r) k.push_back(static_cast<double>(i) / nel);
  for (int i = 0; i <= p; ++i) k.push_back(1.0);
  return make_knots(std::move(k), p);
}

namespace {

// splines.cpp:69-86
void basis_values(const KnotVector& kv, int span, double x, double* out) {
  const int p = kv.degree;
  out[0] = 1.0;
  double left[32], right[32];
  for (int j = 1; j <= p; ++j) {
    left[j] = x - kv.knots[span + 1 - j];
    right[j] = kv.knots[span + j] - x;
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double den = right[r + 1] + left[j - r];
      const double tmp = den > 0.0 ? out[r] / den : 0.0;
      out[r] = saved + right[r + 1] * tmp;
      saved = left[j - r] * tmp;
    }
    out[j] = saved;
  }
}
// splines.cpp:122-171, first derivative
void deriv1_values(const KnotVector& kv, int span, double x, double* out) {
  const int p = kv.degree;
  for (int i = 0; i <= p; ++i) out[i] = 0.0;
  if (p < 1) return;
  const int q = p - 1;
  double low[32];
  KnotVector sub = kv;
  sub.degree = q;
  basis_values(sub, span, x, low);
  const int first = span - p;
  for (int i = 0; i <= p; ++i) {
    const int lo = first + i;
    double c0 = 0.0, c1 = 0.0;
    const double d1 = kv.knots[lo + p] - kv.knots[lo];
    const double d2 = kv.knots[lo + p + 1] - kv.knots[lo + 1];
    if (d1 > 0.0) c0 += 1.0 * p / d1;
    if (d2 > 0.0) c1 -= 1.0 * p / d2;
    double v = 0.0;
    int off = lo - (span - q);
    if (off >= 0 && off <= q) v += c0 * low[off];
    off = lo + 1 - (span - q);
    if (off >= 0 && off <= q) v += c1 * low[off];
    out[i] = v;
  }
}
void check_domain(double x) {
  if (!(x >= 0.0 && x <= 1.0)) throw std::domain_error("eval_basis: parameter outside [0,1]");
}

// Power-basis coefficients (in y = x - knots[span]) of the p+1 basis
// functions nonzero on `span`, by the Cox-de Boor recursion on polynomials
// in long double.  out[fn][k], fn = 0..p  <->  N_{span-p+fn}.
void span_polys(const KnotVector& kv, int span, std::vector<std::vector<long double>>& out) {
  const int p = kv.degree;
  const auto& t = kv.knots;
  const long double ts = t[span];
  std::vector<std::vector<long double>> cur(1, std::vector<long double>(p + 1, 0.0L));
  cur[0][0] = 1.0L;
  for (int k = 1; k <= p; ++k) {
    std::vector<std::vector<long double>> nx(k + 1, std::vector<long double>(p + 1, 0.0L));
    for (int r = 0; r <= k; ++r) {
      const int i = span - k + r;
      if (r >= 1) {  // omega_{i,k} N_{i,k-1}
        const long double den = static_cast<long double>(t[i + k]) - t[i];
        if (den > 0) {
          const long double a = (ts - t[i]) / den, b = 1.0L / den;  // (y + ts - t_i)/den
          const auto& src = cur[r - 1];
          for (int d = p; d >= 0; --d) nx[r][d] += a * src[d] + (d > 0 ? b * src[d - 1] : 0.0L);
        }
      }
      if (r <= k - 1) {  // (1 - omega_{i+1,k}) N_{i+1,k-1}
        const long double den = static_cast<long double>(t[i + k + 1]) - t[i + 1];
        if (den > 0) {
          const long double a = (static_cast<long double>(t[i + k + 1]) - ts) / den, b = -1.0L / den;
          const auto& src = cur[r];
          for (int d = p; d >= 0; --d) nx[r][d] += a * src[d] + (d > 0 ? b * src[d - 1] : 0.0L);
        }
      }
    }
    cur = std::move(nx);
  }
  out = std::move(cur);
}
// substitute y = a + h s: coefficients in s
std::vector<long double> shift_scale(const std::vector<long double>& c, long double a, long double h) {
  const int n = static_cast<int>(c.size());
  std::vector<long double> out(n, 0.0L);
  for (int k = 0; k < n; ++k) {
    // c_k (a + h s)^k = c_k sum_j binom(k,j) a^(k-j) h^j s^j
    long double binom = 1.0L;
    for (int j = 0; j <= k; ++j) {
      out[j] += c[k] * binom * std::pow(a, static_cast<long double>(k - j)) *
                std::pow(h, static_cast<long double>(j));
      binom = binom * (k - j) / (j + 1);
    }
  }
  return out;
}

}  // namespace

V3 Patch::point(int i, int j) const {
  const int idx = i + j * count_u();
  return V3(cw[3 * idx], cw[3 * idx + 1], cw[3 * idx + 2]) / w[idx];
}

// splines.cpp:183-216 -- same expression order, used for the element boxes
Jet eval_patch(const Patch& s, double u, double v) {
  check_domain(u);
  check_domain(v);
  double bu[32], bv[32], du[32], dv[32];
  const int su = s.kv_u.find_span(u), sv = s.kv_v.find_span(v);
  basis_values(s.kv_u, su, u, bu);
  basis_values(s.kv_v, sv, v, bv);
  deriv1_values(s.kv_u, su, u, du);
  deriv1_values(s.kv_v, sv, v, dv);
  const int fu = su - s.kv_u.degree, fv = sv - s.kv_v.degree;
  const int pu = s.kv_u.degree, pv = s.kv_v.degree, ku = s.count_u();
  V3 N, Nu, Nv;
  double W = 0.0, Wu = 0.0, Wv = 0.0;
  for (int j = 0; j <= pv; ++j)
    for (int i = 0; i <= pu; ++i) {
      const int idx = (fu + i) + (fv + j) * ku;
      const double w = s.w[idx];
      const V3 cw(s.cw[3 * idx], s.cw[3 * idx + 1], s.cw[3 * idx + 2]);
      N = N + cw * (bu[i] * bv[j]);
      Nu = Nu + cw * (du[i] * bv[j]);
      Nv = Nv + cw * (bu[i] * dv[j]);
      W += w * bu[i] * bv[j];
      Wu += w * du[i] * bv[j];
      Wv += w * bu[i] * dv[j];
    }
  Jet jet;
  jet.x = N / W;
  jet.du = (Nu - jet.x * Wu) / W;
  jet.dv = (Nv - jet.x * Wv) / W;
  return jet;
}

// ------------------------------------------------------------- geometry
namespace {
void edge_point(int edge, double t, double& u, double& v) {  // geometry.cpp:72-80
  switch (edge) {
    case 0: u = t; v = 0; break;
    case 1: u = 1; v = t; break;
    case 2: u = t; v = 1; break;
    default: u = 0; v = t; break;
  }
}
std::vector<V3> edge_polygon(const Patch& s, int edge) {  // geometry.cpp:17-45
  const int ku = s.count_u(), kv = s.count_v();
  std::vector<V3> poly;
  switch (edge) {
    case 0: for (int i = 0; i < ku; ++i) poly.push_back(s.point(i, 0)); break;
    case 1: for (int j = 0; j < kv; ++j) poly.push_back(s.point(ku - 1, j)); break;
    case 2: for (int i = 0; i < ku; ++i) poly.push_back(s.point(i, kv - 1)); break;
    default: for (int j = 0; j < kv; ++j) poly.push_back(s.point(0, j)); break;
  }
  return poly;
}
bool polys_match(const std::vector<V3>& a, const std::vector<V3>& b, bool& rev) {
  if (a.size() != b.size()) return false;
  const int n = static_cast<int>(a.size());
  double fwd = 0, bwd = 0;
  for (int i = 0; i < n; ++i) {
    fwd = std::max(fwd, norm(a[i] - b[i]));
    bwd = std::max(bwd, norm(a[i] - b[n - 1 - i]));
  }
  if (fwd <= 1e-9) { rev = false; return true; }
  if (bwd <= 1e-9) { rev = true; return true; }
  return false;
}
V3 corner_ctrl(const Patch& s, int corner) {
  const int i = (corner == 1 || corner == 3) ? s.count_u() - 1 : 0;
  const int j = (corner >= 2) ? s.count_v() - 1 : 0;
  return s.point(i, j);
}
struct FrameLite {
  V3 x, normal;
  double sqrt_g;
};
FrameLite frame(const Patch& p, double u, double v) {  // geometry.cpp:167-176
  const Jet j = eval_patch(p, u, v);
  FrameLite f;
  f.x = j.x;
  f.normal = cross(j.du, j.dv);
  f.sqrt_g = norm(f.normal);
  return f;
}
}  // namespace

// geometry.cpp:88-163
Geometry::Geometry(std::vector<Patch> patches) : patches_(std::move(patches)) {
  if (patches_.empty()) throw std::invalid_argument("Geometry: no patches");
  for (const auto& p : patches_) {
    const int n = p.count_u() * p.count_v();
    if (static_cast<int>(p.w.size()) != n || static_cast<int>(p.cw.size()) != 3 * n)
      throw std::invalid_argument("PatchSurface: control grid does not match basis counts");
    for (double x : p.w)
      if (!(x > 0.0)) throw std::invalid_argument("PatchSurface: weights must be strictly positive");
  }
  const int m = patch_count();
  std::vector<int> paired(4 * m, 0);
  for (int a = 0; a < m; ++a)
    for (int ea = 0; ea < 4; ++ea) {
      const auto pa = edge_polygon(patches_[a], ea);
      for (int b = a; b < m; ++b)
        for (int eb = (b == a ? ea + 1 : 0); eb < 4; ++eb) {
          bool rev = false;
          if (polys_match(pa, edge_polygon(patches_[b], eb), rev)) {
            edges_.push_back({a, ea, b, eb, rev});
            if (++paired[4 * a + ea] > 1 || ++paired[4 * b + eb] > 1)
              throw std::runtime_error("Geometry: three or more coincident edges");
          }
        }
    }
  for (int a = 0; a < m; ++a)
    for (int ca = 0; ca < 4; ++ca) {
      const V3 xa = corner_ctrl(patches_[a], ca);
      for (int b = a; b < m; ++b)
        for (int cb = (b == a ? ca + 1 : 0); cb < 4; ++cb)
          if (norm(xa - corner_ctrl(patches_[b], cb)) <= 1e-9) vertices_.push_back({a, ca, b, cb});
    }
  for (int p = 0; p < m; ++p)
    for (int i = 0; i < 5; ++i)
      for (int j = 0; j < 5; ++j)
        if (frame(patches_[p], i / 4.0, j / 4.0).sqrt_g < 1e-12)
          throw std::runtime_error("Geometry: degenerate parametrization on patch " + std::to_string(p));
  if (static_cast<int>(edges_.size()) == 2 * m) {
    V3 centroid;
    int n = 0;
    for (int p = 0; p < m; ++p)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          centroid = centroid + frame(patches_[p], 0.25 + 0.25 * i, 0.25 + 0.25 * j).x;
          ++n;
        }
    centroid = centroid / n;
    for (int p = 0; p < m; ++p)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const FrameLite f = frame(patches_[p], 0.25 + 0.25 * i, 0.25 + 0.25 * j);
          if (dot(f.normal, f.x - centroid) <= 0.0)
            throw std::runtime_error("Geometry: normal of patch " + std::to_string(p) +
                                     " is not outward pointing");
        }
  }
}

double Geometry::check_matching() const {  // geometry.cpp:178-195
  double worst = 0;
  for (const auto& e : edges_) {
    double dev = 0;
    for (int k = 0; k < 17; ++k) {
      const double t = k / 16.0;
      const double tb = e.reversed ? 1.0 - t : t;
      double ua, va, ub, vb;
      edge_point(e.edge_a, t, ua, va);
      edge_point(e.edge_b, tb, ub, vb);
      dev = std::max(dev, norm(eval_patch(patches_[e.patch_a], ua, va).x -
                               eval_patch(patches_[e.patch_b], ub, vb).x));
    }
    if (dev > 1e-9) worst = std::max(worst, dev);
  }
  return worst;
}

// --------------------------------------------------------------- shapes
namespace {
// bivariate power-basis polynomial, column-major (shapes.cpp:34-58)
struct Poly2 {
  int r = 1, c = 1;
  std::vector<double> a;
  Poly2() : a(1, 0.0) {}
  Poly2(int rr, int cc) : r(rr), c(cc), a(rr * cc, 0.0) {}
  double& operator()(int i, int j) { return a[i + r * j]; }
  double operator()(int i, int j) const { return a[i + r * j]; }
};
Poly2 pscale(const Poly2& x, double s) {
  Poly2 y = x;
  for (auto& v : y.a) v = v * s;
  return y;
}
Poly2 pneg(const Poly2& x) {
  Poly2 y = x;
  for (auto& v : y.a) v = -v;
  return y;
}
Poly2 pmul(const Poly2& a, const Poly2& b) {
  Poly2 c(a.r + b.r - 1, a.c + b.c - 1);
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j)
      for (int k = 0; k < b.r; ++k)
        for (int l = 0; l < b.c; ++l) c(i + k, j + l) += a(i, j) * b(k, l);
  return c;
}
Poly2 padd(const Poly2& a, const Poly2& b) {
  Poly2 c(std::max(a.r, b.r), std::max(a.c, b.c));
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i) c(i, j) = a(i, j);
  for (int j = 0; j < b.c; ++j)
    for (int i = 0; i < b.r; ++i) c(i, j) += b(i, j);
  return c;
}
double binom(int n, int k) {
  double r = 1;
  for (int i = 0; i < k; ++i) r = r * (n - i) / (i + 1);
  return r;
}
void power_to_bernstein(const double* a, int na, int n, double* c) {
  for (int j = 0; j <= n; ++j) c[j] = 0.0;
  for (int j = 0; j <= n; ++j)
    for (int k = 0; k <= j && k < na; ++k) c[j] += a[k] * binom(j, k) / binom(n, k);
}
V3 normalized(const V3& a) {
  const double z = dot(a, a);
  return z > 0 ? a / std::sqrt(z) : a;
}
}  // namespace

std::shared_ptr<Geometry> make_square() {  // shapes.cpp:9-30 (p = 1)
  Patch s;
  s.kv_u = make_uniform_knots(1, 0, 1);
  s.kv_v = make_uniform_knots(1, 0, 1);
  s.cw.resize(12);
  s.w.assign(4, 1.0);
  for (int j = 0; j < 2; ++j)
    for (int i = 0; i < 2; ++i) {
      const V3 x = V3(0, 0, 0) + V3(1, 0, 0) * double(i) + V3(0, 1, 0) * double(j);
      for (int c = 0; c < 3; ++c) s.cw[3 * (i + 2 * j) + c] = x[c];
    }
  return std::make_shared<Geometry>(std::vector<Patch>{s});
}

// shapes.cpp:87-205
std::shared_ptr<Geometry> make_sphere(double radius, const V3& center) {
  if (radius <= 0) throw std::invalid_argument("make_sphere: radius must be positive");
  const double s = 1.0 / std::sqrt(3.0);
  struct Face {
    V3 a;
    V3 c[4];
  };
  const Face faces[6] = {
      {{1, 0, 0}, {{1, -1, -1}, {1, 1, -1}, {1, -1, 1}, {1, 1, 1}}},
      {{-1, 0, 0}, {{-1, -1, -1}, {-1, -1, 1}, {-1, 1, -1}, {-1, 1, 1}}},
      {{0, 1, 0}, {{-1, 1, -1}, {-1, 1, 1}, {1, 1, -1}, {1, 1, 1}}},
      {{0, -1, 0}, {{-1, -1, -1}, {1, -1, -1}, {-1, -1, 1}, {1, -1, 1}}},
      {{0, 0, 1}, {{-1, -1, 1}, {1, -1, 1}, {-1, 1, 1}, {1, 1, 1}}},
      {{0, 0, -1}, {{-1, -1, -1}, {-1, 1, -1}, {1, -1, -1}, {1, 1, -1}}},
  };
  std::vector<Patch> patches;
  for (const auto& face : faces) {
    const V3 a = face.a;
    const V3 ref = std::abs(a[0]) < 0.9 ? V3(1, 0, 0) : V3(0, 1, 0);
    const V3 e1 = normalized(cross(a, ref));
    const V3 e2 = cross(a, e1);
    V3 C[4];
    for (int i = 0; i < 4; ++i) C[i] = face.c[i] * s;
    // arc_h + project (shapes.cpp:78-85,116-125)
    auto arc2d = [&](const V3& A, const V3& B) {
      const double c = dot(A, B);
      const double w = std::sqrt((1.0 + c) / 2.0);
      const V3 M = (A + B) / (1.0 + c);
      const double h[3][4] = {{A[0], A[1], A[2], 1.0}, {w * M[0], w * M[1], w * M[2], w},
                              {B[0], B[1], B[2], 1.0}};
      std::array<V3, 3> out;
      for (int k = 0; k < 3; ++k) {
        const V3 x(h[k][0], h[k][1], h[k][2]);
        out[k] = V3(dot(e1, x), dot(e2, x), h[k][3] + dot(a, x));
      }
      return out;
    };
    const auto bottom = arc2d(C[0], C[1]);
    const auto top = arc2d(C[2], C[3]);
    const auto left = arc2d(C[0], C[2]);
    const auto right = arc2d(C[1], C[3]);
    Poly2 one(1, 1);
    one(0, 0) = 1.0;
    Poly2 u(2, 1), v(1, 2);
    u(1, 0) = 1;
    v(0, 1) = 1;
    const Poly2 mu = padd(one, pneg(u)), mv = padd(one, pneg(v));
    auto bern2 = [&](const Poly2& t, int k) {
      const Poly2 mt = padd(one, pneg(t));
      if (k == 0) return pmul(mt, mt);
      if (k == 1) return pmul(pmul(pscale(one, 2.0), t), mt);
      return pmul(t, t);
    };
    Poly2 P[3];
    for (int c = 0; c < 3; ++c) {
      Poly2 acc(1, 1);
      for (int k = 0; k < 3; ++k) {
        acc = padd(acc, pscale(pmul(mv, bern2(u, k)), bottom[k][c]));
        acc = padd(acc, pscale(pmul(v, bern2(u, k)), top[k][c]));
        acc = padd(acc, pscale(pmul(mu, bern2(v, k)), left[k][c]));
        acc = padd(acc, pscale(pmul(u, bern2(v, k)), right[k][c]));
      }
      acc = padd(acc, pscale(pmul(mu, mv), -bottom[0][c]));
      acc = padd(acc, pscale(pmul(u, mv), -bottom[2][c]));
      acc = padd(acc, pscale(pmul(mu, v), -top[0][c]));
      acc = padd(acc, pscale(pmul(u, v), -top[2][c]));
      P[c] = acc;
    }
    const Poly2 xi = P[0], eta = P[1], om = P[2];
    const Poly2 xi2 = pmul(xi, xi), eta2 = pmul(eta, eta), om2 = pmul(om, om);
    const Poly2 mone = pneg(one);
    const Poly2 radial = padd(om2, padd(pmul(xi2, mone), pmul(eta2, mone)));
    Poly2 H[4];
    for (int c = 0; c < 3; ++c) {
      Poly2 acc = pscale(pmul(pscale(pmul(xi, om), 2.0), one), e1[c]);
      acc = padd(acc, pscale(pmul(eta, om), 2.0 * e2[c]));
      acc = padd(acc, pscale(radial, a[c]));
      H[c] = acc;
    }
    H[3] = padd(om2, padd(xi2, eta2));
    Patch patch;
    patch.kv_u = make_uniform_knots(4, 0, 1);
    patch.kv_v = make_uniform_knots(4, 0, 1);
    double net[4][25];
    for (int c = 0; c < 4; ++c) {
      double full[5][5] = {};
      for (int j = 0; j < H[c].c; ++j)
        for (int i = 0; i < H[c].r; ++i) full[i][j] = H[c](i, j);
      double tmp[5][5], col[5], b[5];
      for (int j = 0; j < 5; ++j) {
        for (int i = 0; i < 5; ++i) col[i] = full[i][j];
        power_to_bernstein(col, 5, 4, b);
        for (int i = 0; i < 5; ++i) tmp[i][j] = b[i];
      }
      for (int i = 0; i < 5; ++i) {
        power_to_bernstein(tmp[i], 5, 4, b);
        for (int j = 0; j < 5; ++j) full[i][j] = b[j];
      }
      for (int j = 0; j < 5; ++j)
        for (int i = 0; i < 5; ++i) net[c][i + 5 * j] = full[i][j];
    }
    patch.w.resize(25);
    patch.cw.resize(75);
    for (int i = 0; i < 25; ++i) {
      patch.w[i] = net[3][i];
      if (patch.w[i] <= 0.0) throw std::logic_error("make_sphere: nonpositive weight in lifted patch");
      for (int c = 0; c < 3; ++c) patch.cw[3 * i + c] = radius * net[c][i] + center[c] * net[3][i];
    }
    patches.push_back(std::move(patch));
  }
  return std::make_shared<Geometry>(std::move(patches));
}

// ------------------------------------------------------- discretization
namespace {
struct SignedUnionFind {  // spaces.cpp:10-38
  std::vector<int> parent;
  std::vector<double> sign;
  explicit SignedUnionFind(int n) : parent(n), sign(n, 1.0) {
    for (int i = 0; i < n; ++i) parent[i] = i;
  }
  std::pair<int, double> find(int i) {
    if (parent[i] == i) return {i, 1.0};
    auto [r, s] = find(parent[i]);
    parent[i] = r;
    sign[i] *= s;
    return {r, sign[i]};
  }
  void unite(int a, int b, double rel) {
    auto [ra, sa] = find(a);
    auto [rb, sb] = find(b);
    if (ra == rb) {
      if (sb != rel * sa) throw std::runtime_error("Discretization: inconsistent edge orientation gluing");
      return;
    }
    parent[rb] = ra;
    sign[rb] = rel * sa / sb;
  }
};
bool element_on_edge(int edge, int ix, int iy, int n) {
  switch (edge) {
    case 0: return iy == 0;
    case 1: return ix == n - 1;
    case 2: return iy == n - 1;
    case 3: return ix == 0;
  }
  return false;
}
int grid_pos_on_edge(int edge, int ix, int iy) { return (edge == 0 || edge == 2) ? ix : iy; }
int edge_end_corner(int edge, int end) {
  static const int tbl[4][2] = {{0, 1}, {1, 3}, {2, 3}, {0, 2}};
  return tbl[edge][end];
}
bool element_at_corner(int corner, int ix, int iy, int n) {
  const int cx = (corner == 1 || corner == 3) ? n - 1 : 0;
  const int cy = (corner >= 2) ? n - 1 : 0;
  return ix == cx && iy == cy;
}
SquareMap map_bottom_to_edge(int edge, bool reversed) {  // quadrature.cpp:52-63
  switch (edge) {
    case 0: return {false, reversed, false};
    case 1: return {true, true, reversed};
    case 2: return {false, reversed, true};
    default: return {true, false, reversed};
  }
}
SquareMap map_origin_to_corner(int corner) {  // quadrature.cpp:65-73
  switch (corner) {
    case 0: return {false, false, false};
    case 1: return {false, true, false};
    case 2: return {false, false, true};
    default: return {false, true, true};
  }
}
}  // namespace

// spaces.cpp:71-115
Discretization::Discretization(std::shared_ptr<const Geometry> g, int kind, cplx kappa, int degree,
                               int rep, int level)
    : geom_(std::move(g)), kind_(kind), kappa_(kappa), degree_(degree), rep_(rep), level_(level) {
  if (!geom_) throw std::invalid_argument("Discretization: null geometry");
  if (kind < kLaplace || kind > kMaxwell) throw std::invalid_argument("Discretization: unknown kind");
  if (kind == kMaxwell && kappa == cplx(0, 0))
    throw std::invalid_argument("Pde: Maxwell requires a nonzero wavenumber");
  if (level < 0) throw std::invalid_argument("Discretization: negative level");
  if (level > 14) throw std::invalid_argument("Discretization: level too large");
  if (kind == kMaxwell) {
    if (degree < 1) throw std::invalid_argument("Discretization: Maxwell requires degree P >= 1");
    if (rep != 1)
      throw std::invalid_argument(
          "Discretization: the div-conforming space supports knot repetition 1 only");
  } else if (degree < 0) {
    throw std::invalid_argument("Discretization: negative degree");
  }
  if (rep < 1 || rep > std::max(degree, 0) + 1)
    throw std::invalid_argument("Discretization: knot repetition out of range");
  if (geom_->check_matching() > 0)
    throw std::runtime_error("Discretization: geometry fails the matching condition");
  const int m = geom_->patch_count();
  cross_edges_.assign(m, std::vector<std::vector<CrossEdge>>(m));
  cross_corners_.assign(m, std::vector<std::vector<CrossCorner>>(m));
  for (const auto& e : geom_->edges()) {
    cross_edges_[e.patch_a][e.patch_b].push_back({e.edge_a, e.edge_b, e.reversed});
    cross_edges_[e.patch_b][e.patch_a].push_back({e.edge_b, e.edge_a, e.reversed});
  }
  for (const auto& v : geom_->vertices()) {
    cross_corners_[v.patch_a][v.patch_b].push_back({v.corner_a, v.corner_b});
    cross_corners_[v.patch_b][v.patch_a].push_back({v.corner_b, v.corner_a});
  }
  build_elements();
  if (kind == kMaxwell)
    build_maxwell();
  else
    build_scalar();
  build_cells();
  build_tables();
}

void Discretization::build_elements() {  // spaces.cpp:117-147
  const int n = 1 << level_;
  const double h = 1.0 / n;
  const int m = geom_->patch_count();
  epp_ = n * n;
  elements_.resize(static_cast<size_t>(m) * epp_);
  const int ns = degree_ + 2;
#pragma omp parallel for schedule(static)
  for (int idx = 0; idx < m * epp_; ++idx) {
    const int p = idx / epp_, r = idx % epp_, iy = r / n, ix = r % n;
    Element el;
    el.patch = p;
    el.ix = ix;
    el.iy = iy;
    el.h = h;
    el.ox = ix * h;
    el.oy = iy * h;
    el.box.set_empty();
    for (int a = 0; a < ns; ++a)
      for (int b = 0; b < ns; ++b) {
        const double u = el.ox + h * a / (ns - 1.0);
        const double v = el.oy + h * b / (ns - 1.0);
        el.box.extend(eval_patch(geom_->patch(p), u, v).x);
      }
    double c[3], half[3];
    for (int k = 0; k < 3; ++k) c[k] = (el.box.mn[k] + el.box.mx[k]) / 2.0;
    for (int k = 0; k < 3; ++k) half[k] = 1.1 * (el.box.mx[k] - c[k]);
    for (int k = 0; k < 3; ++k) {
      el.box.mn[k] = c[k] - half[k];
      el.box.mx[k] = c[k] + half[k];
    }
    elements_[idx] = el;
  }
}

void Discretization::build_scalar() {  // spaces.cpp:149-176
  if (degree_ == 0)
    scalar_kv_ = make_uniform_knots(0, level_, 1);
  else
    scalar_kv_ = make_uniform_knots(degree_ - 1, level_, std::min(rep_, degree_));
  const int k = scalar_kv_.size();
  const int q = scalar_kv_.degree;
  scalar_q_ = q;
  n_local_ = (q + 1) * (q + 1);
  const int per_patch = k * k;
  n_dofs_ = geom_->patch_count() * per_patch;
  const int ne = element_count();
  l2g_.resize(static_cast<size_t>(ne) * n_local_);
  lsign_.assign(static_cast<size_t>(ne) * n_local_, 1.0);
  for (int e = 0; e < ne; ++e) {
    const auto& el = elements_[e];
    const int fu = scalar_kv_.find_span(el.ox + 0.5 * el.h) - q;
    const int fv = scalar_kv_.find_span(el.oy + 0.5 * el.h) - q;
    int l = 0;
    for (int j = 0; j <= q; ++j)
      for (int i = 0; i <= q; ++i, ++l)
        l2g_[static_cast<size_t>(e) * n_local_ + l] = el.patch * per_patch + (fu + i) + k * (fv + j);
  }
}

void Discretization::build_maxwell() {  // spaces.cpp:178-255
  const int P = degree_;
  vec_kv_p_ = make_uniform_knots(P, level_, 1);
  vec_kv_q_ = make_uniform_knots(P - 1, level_, 1);
  const int kp = vec_kv_p_.size(), kq = vec_kv_q_.size();
  const int m = geom_->patch_count();
  const int per_block = kp * kq, per_patch = 2 * per_block, n_raw = m * per_patch;
  auto raw_u = [&](int patch, int i, int j) { return patch * per_patch + i + kp * j; };
  auto raw_v = [&](int patch, int i, int j) { return patch * per_patch + per_block + i + kq * j; };
  auto strip = [&](int patch, int edge, int s) -> std::pair<int, double> {
    switch (edge) {
      case 0: return {raw_v(patch, s, 0), -1.0};
      case 1: return {raw_u(patch, kp - 1, s), +1.0};
      case 2: return {raw_v(patch, s, kp - 1), +1.0};
      default: return {raw_u(patch, 0, s), -1.0};
    }
  };
  SignedUnionFind uf(n_raw);
  for (const auto& e : geom_->edges())
    for (int s = 0; s < kq; ++s) {
      const int sb = e.reversed ? kq - 1 - s : s;
      const auto [ra, ea] = strip(e.patch_a, e.edge_a, s);
      const auto [rb, eb] = strip(e.patch_b, e.edge_b, sb);
      uf.unite(ra, rb, -ea * eb);
    }
  std::vector<int> glob(n_raw, -1);
  std::vector<double> gsign(n_raw, 1.0);
  int next = 0;
  for (int i = 0; i < n_raw; ++i) {
    auto [r, s] = uf.find(i);
    if (glob[r] < 0) glob[r] = next++;
    glob[i] = glob[r];
    gsign[i] = s;
  }
  n_dofs_ = next;
  n_local_ = 2 * (P + 1) * P;
  const int ne = element_count();
  l2g_.resize(static_cast<size_t>(ne) * n_local_);
  lsign_.resize(static_cast<size_t>(ne) * n_local_);
  for (int e = 0; e < ne; ++e) {
    const auto& el = elements_[e];
    const double midu = el.ox + 0.5 * el.h, midv = el.oy + 0.5 * el.h;
    const int fpu = vec_kv_p_.find_span(midu) - P, fpv = vec_kv_p_.find_span(midv) - P;
    const int fqu = vec_kv_q_.find_span(midu) - (P - 1), fqv = vec_kv_q_.find_span(midv) - (P - 1);
    int l = 0;
    for (int j = 0; j < P; ++j)
      for (int i = 0; i <= P; ++i, ++l) {
        const int r = raw_u(el.patch, fpu + i, fqv + j);
        l2g_[static_cast<size_t>(e) * n_local_ + l] = glob[r];
        lsign_[static_cast<size_t>(e) * n_local_ + l] = gsign[r];
      }
    for (int j = 0; j <= P; ++j)
      for (int i = 0; i < P; ++i, ++l) {
        const int r = raw_v(el.patch, fqu + i, fpv + j);
        l2g_[static_cast<size_t>(e) * n_local_ + l] = glob[r];
        lsign_[static_cast<size_t>(e) * n_local_ + l] = gsign[r];
      }
  }
}

// Patch knot-span cells in power form; every element must lie in one cell.
void Discretization::build_cells() {
  const int np = geom_->patch_count();
  std::vector<int> cell_base(np + 1, 0);
  geom_degree_ = 0;
  for (int p = 0; p < np; ++p) {
    const Patch& s = geom_->patch(p);
    if (s.kv_u.degree > kMaxGeomDeg || s.kv_v.degree > kMaxGeomDeg)
      throw std::invalid_argument("B200 H2: geometry degree > 4 is not supported");
    geom_degree_ = std::max({geom_degree_, s.kv_u.degree, s.kv_v.degree});
    const int nsu = s.kv_u.size() - s.kv_u.degree, nsv = s.kv_v.size() - s.kv_v.degree;
    cell_base[p + 1] = cell_base[p] + nsu * nsv;  // spans degree..size-1 (some may be empty)
  }
  cells_.assign(cell_base[np], GeomCell{});
  for (int p = 0; p < np; ++p) {
    const Patch& s = geom_->patch(p);
    const int pu = s.kv_u.degree, pv = s.kv_v.degree;
    const int nsu = s.kv_u.size() - pu, nsv = s.kv_v.size() - pv;
    for (int a = 0; a < nsu; ++a)
      for (int b = 0; b < nsv; ++b) {
        const int su = pu + a, sv = pv + b;
        GeomCell& cell = cells_[cell_base[p] + a * nsv + b];
        cell.u0 = s.kv_u.knots[su];
        cell.v0 = s.kv_v.knots[sv];
        if (!(s.kv_u.knots[su + 1] > s.kv_u.knots[su]) || !(s.kv_v.knots[sv + 1] > s.kv_v.knots[sv])) continue;
        std::vector<std::vector<long double>> nu, nv;
        span_polys(s.kv_u, su, nu);
        span_polys(s.kv_v, sv, nv);
        const int fu = su - pu, fv = sv - pv, ku = s.count_u();
        for (int c = 0; c < 4; ++c)
          for (int l = 0; l <= pv; ++l)
            for (int k = 0; k <= pu; ++k) {
              long double acc = 0.0L;
              for (int j = 0; j <= pv; ++j)
                for (int i = 0; i <= pu; ++i) {
                  const int idx = (fu + i) + (fv + j) * ku;
                  const double val = c < 3 ? s.cw[3 * idx + c] : s.w[idx];
                  acc += nu[i][k] * nv[j][l] * static_cast<long double>(val);
                }
              cell.coef[c][l][k] = static_cast<double>(acc);
            }
      }
  }
  const int ne = element_count();
  element_cell_.resize(ne);
  for (int e = 0; e < ne; ++e) {
    const Element& el = elements_[e];
    const Patch& s = geom_->patch(el.patch);
    const int su = s.kv_u.find_span(el.ox + 0.5 * el.h), sv = s.kv_v.find_span(el.oy + 0.5 * el.h);
    if (el.ox < s.kv_u.knots[su] || el.ox + el.h > s.kv_u.knots[su + 1] || el.oy < s.kv_v.knots[sv] ||
        el.oy + el.h > s.kv_v.knots[sv + 1])
      throw std::invalid_argument("B200 H2: element straddles a geometry knot span");
    const int nsv = s.kv_v.size() - s.kv_v.degree;
    element_cell_[e] = cell_base[el.patch] + (su - s.kv_u.degree) * nsv + (sv - s.kv_v.degree);
  }
}

// 1D element-local basis polynomials for every grid position
void Discretization::build_tables() {
  const int n = 1 << level_;
  const double h = 1.0 / n;
  auto fill = [&](const KnotVector& kv, std::vector<double>& tab) {
    const int p = kv.degree;
    tab.assign(static_cast<size_t>(n) * (p + 1) * (p + 1), 0.0);
    for (int pos = 0; pos < n; ++pos) {
      const double ox = pos * h;
      const int span = kv.find_span(ox + 0.5 * h);
      std::vector<std::vector<long double>> polys;
      span_polys(kv, span, polys);
      for (int fn = 0; fn <= p; ++fn) {
        const auto loc = shift_scale(polys[fn], static_cast<long double>(ox) - kv.knots[span], h);
        for (int k = 0; k <= p; ++k) tab[(static_cast<size_t>(pos) * (p + 1) + fn) * (p + 1) + k] = static_cast<double>(loc[k]);
      }
    }
  };
  if (kind_ == kMaxwell) {
    fill(vec_kv_p_, tab_p_);
    fill(vec_kv_q_, tab_q_);
  } else {
    fill(scalar_kv_, tab_s_);
  }
}

// spaces.cpp:309-394
PairInfo Discretization::classify_pair(int ea, int eb) const {
  PairInfo info;
  if (ea == eb) {
    info.cls = kCoincident;
    return info;
  }
  const auto& a = elements_[ea];
  const auto& b = elements_[eb];
  const int n = 1 << level_;
  int best = 0;
  PairInfo cand;
  if (a.patch == b.patch) {
    const int dx = b.ix - a.ix, dy = b.iy - a.iy;
    if (std::abs(dx) <= 1 && std::abs(dy) <= 1) {
      if (std::abs(dx) + std::abs(dy) == 1) {
        int edge_a, edge_b;
        if (dx == 1) { edge_a = 1; edge_b = 3; }
        else if (dx == -1) { edge_a = 3; edge_b = 1; }
        else if (dy == 1) { edge_a = 2; edge_b = 0; }
        else { edge_a = 0; edge_b = 2; }
        cand.cls = kEdge;
        cand.map_a = map_bottom_to_edge(edge_a, false);
        cand.map_b = map_bottom_to_edge(edge_b, false);
        best = 2;
      } else {
        const int ca = (dx > 0 ? 1 : 0) + (dy > 0 ? 2 : 0);
        const int cb = (dx > 0 ? 0 : 1) + (dy > 0 ? 0 : 2);
        cand.cls = kVertex;
        cand.map_a = map_origin_to_corner(ca);
        cand.map_b = map_origin_to_corner(cb);
        best = 1;
      }
    }
  }
  if (best < 2) {
    for (const auto& ce : cross_edges_[a.patch][b.patch]) {
      if (!element_on_edge(ce.edge_a, a.ix, a.iy, n)) continue;
      if (!element_on_edge(ce.edge_b, b.ix, b.iy, n)) continue;
      const int sa = grid_pos_on_edge(ce.edge_a, a.ix, a.iy);
      const int sb_raw = grid_pos_on_edge(ce.edge_b, b.ix, b.iy);
      const int sb = ce.reversed ? n - 1 - sb_raw : sb_raw;
      if (sa == sb) {
        cand.cls = kEdge;
        cand.map_a = map_bottom_to_edge(ce.edge_a, false);
        cand.map_b = map_bottom_to_edge(ce.edge_b, ce.reversed);
        best = 2;
        break;
      }
      if (std::abs(sa - sb) == 1 && best < 1) {
        const int end_a = (sb > sa) ? 1 : 0;
        const int end_b_pos = ce.reversed ? end_a : 1 - end_a;
        cand.cls = kVertex;
        cand.map_a = map_origin_to_corner(edge_end_corner(ce.edge_a, end_a));
        cand.map_b = map_origin_to_corner(edge_end_corner(ce.edge_b, end_b_pos));
        best = 1;
      }
    }
  }
  if (best < 1 && a.patch != b.patch) {
    for (const auto& cc : cross_corners_[a.patch][b.patch]) {
      if (element_at_corner(cc.corner_a, a.ix, a.iy, n) && element_at_corner(cc.corner_b, b.ix, b.iy, n)) {
        cand.cls = kVertex;
        cand.map_a = map_origin_to_corner(cc.corner_a);
        cand.map_b = map_origin_to_corner(cc.corner_b);
        best = 1;
        break;
      }
    }
  }
  if (best > 0) info = cand;
  return info;
}

void Discretization::flatten_topology(std::vector<int>& edge_rs, std::vector<int>& edges, std::vector<int>& corner_rs,
                                      std::vector<int>& corners) const {
  const int np = geom_->patch_count();
  edge_rs.assign(np * np + 1, 0);
  corner_rs.assign(np * np + 1, 0);
  edges.clear();
  corners.clear();
  for (int a = 0; a < np; ++a)
    for (int b = 0; b < np; ++b) {
      for (const auto& ce : cross_edges_[a][b]) {
        edges.push_back(ce.edge_a);
        edges.push_back(ce.edge_b);
        edges.push_back(ce.reversed ? 1 : 0);
      }
      for (const auto& cc : cross_corners_[a][b]) {
        corners.push_back(cc.corner_a);
        corners.push_back(cc.corner_b);
      }
      edge_rs[a * np + b + 1] = static_cast<int>(edges.size() / 3);
      corner_rs[a * np + b + 1] = static_cast<int>(corners.size() / 2);
    }
}

void Discretization::singular_items(const unsigned char* owned, SingList out[4]) const {
  const int ne = element_count(), n = 1 << level_, np = geometry().patch_count();
  // patches sharing an edge / a corner with each patch
  std::vector<std::vector<int>> edge_nb(np), corner_nb(np);
  for (int p = 0; p < np; ++p)
    for (int q = 0; q < np; ++q) {
      if (!cross_edges_[p][q].empty()) edge_nb[p].push_back(q);
      if (!cross_corners_[p][q].empty()) corner_nb[p].push_back(q);
    }
  auto edge_element = [&](int patch, int edge, int s) {  // element at position s along a patch edge
    switch (edge) {
      case 0: return element_index(patch, s, 0);
      case 1: return element_index(patch, n - 1, s);
      case 2: return element_index(patch, s, n - 1);
      default: return element_index(patch, 0, s);
    }
  };
  auto corner_element = [&](int patch, int corner) {
    return element_index(patch, (corner == 1 || corner == 3) ? n - 1 : 0, corner >= 2 ? n - 1 : 0);
  };
  int nt = 1;
#ifdef _OPENMP
  nt = omp_get_max_threads();
#endif
  std::vector<SingList> part(static_cast<size_t>(nt) * 4);
#pragma omp parallel num_threads(nt)
  {
    int t = 0;
#ifdef _OPENMP
    t = omp_get_thread_num();
#endif
    const int e0 = static_cast<int>(static_cast<long long>(ne) * t / nt);
    const int e1 = static_cast<int>(static_cast<long long>(ne) * (t + 1) / nt);
    std::vector<int> cand;
    for (int ea = e0; ea < e1; ++ea) {
      const Element& a = elements_[ea];
      cand.clear();
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          const int x = a.ix + dx, y = a.iy + dy;
          if (x >= 0 && x < n && y >= 0 && y < n) cand.push_back(element_index(a.patch, x, y));
        }
      for (int pb : edge_nb[a.patch])
        for (const auto& ce : cross_edges_[a.patch][pb]) {
          if (!element_on_edge(ce.edge_a, a.ix, a.iy, n)) continue;
          const int sa = grid_pos_on_edge(ce.edge_a, a.ix, a.iy);
          for (int sb = std::max(0, sa - 1); sb <= std::min(n - 1, sa + 1); ++sb)
            cand.push_back(edge_element(pb, ce.edge_b, ce.reversed ? n - 1 - sb : sb));
        }
      for (int pb : corner_nb[a.patch])
        for (const auto& cc : cross_corners_[a.patch][pb])
          if (element_at_corner(cc.corner_a, a.ix, a.iy, n)) cand.push_back(corner_element(pb, cc.corner_b));
      std::sort(cand.begin(), cand.end());
      cand.erase(std::unique(cand.begin(), cand.end()), cand.end());
      for (int eb : cand) {
        if (eb < ea || (owned && !owned[ea] && !owned[eb])) continue;
        const PairInfo info = classify_pair(ea, eb);
        if (info.cls == kFar) continue;
        SingList& L = part[static_cast<size_t>(t) * 4 + info.cls];
        L.ea.push_back(ea);
        L.eb.push_back(eb);
        L.map_a.push_back(static_cast<uint8_t>(info.map_a.bits()));
        L.map_b.push_back(static_cast<uint8_t>(info.map_b.bits()));
      }
    }
  }
  for (int c = 1; c <= 3; ++c) {
    SingList& L = out[c];
    L = SingList{};
    for (int t = 0; t < nt; ++t) {
      const SingList& S = part[static_cast<size_t>(t) * 4 + c];
      L.ea.insert(L.ea.end(), S.ea.begin(), S.ea.end());
      L.eb.insert(L.eb.end(), S.eb.begin(), S.eb.end());
      L.map_a.insert(L.map_a.end(), S.map_a.begin(), S.map_a.end());
      L.map_b.insert(L.map_b.end(), S.map_b.begin(), S.map_b.end());
    }
  }
}

// ---------------------------------------------------------- quadrature
void gauss_rule(int n, std::vector<double>& nodes, std::vector<double>& weights) {  // quadrature.cpp:15-50
  if (n < 1 || n > 64) throw std::invalid_argument("gauss_rule: order out of range");
  nodes.assign(n, 0.0);
  weights.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double dp = 0;
    for (int it = 0; it < 100; ++it) {
      double p0 = 1.0, p1 = x;
      for (int k = 2; k <= n; ++k) {
        const double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
        p0 = p1;
        p1 = p2;
      }
      dp = n * (x * p1 - p0) / (x * x - 1.0);
      const double dx = p1 / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    nodes[n - 1 - i] = 0.5 * (1.0 + x);
    weights[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
  }
}
std::vector<double> cheb_nodes(int m) {  // h2.cpp:13-17
  std::vector<double> x(m);
  for (int k = 0; k < m; ++k) x[k] = 0.5 * (1.0 - std::cos(M_PI * k / (m - 1)));
  return x;
}
void lagrange_all(const std::vector<double>& nodes, double x, double* out) {  // h2.cpp:19-45
  const int m = static_cast<int>(nodes.size());
  for (int k = 0; k < m; ++k) out[k] = 0.0;
  for (int k = 0; k < m; ++k)
    if (x == nodes[k]) {
      out[k] = 1.0;
      return;
    }
  double denom = 0;
  for (int k = 0; k < m; ++k) {
    double bw = (k % 2 == 0) ? 1.0 : -1.0;
    if (k == 0 || k == m - 1) bw *= 0.5;
    out[k] = bw / (x - nodes[k]);
    denom += out[k];
  }
  for (int k = 0; k < m; ++k) out[k] /= denom;
}

// ------------------------------------------------------------ H2 plan
void check_h2_options(const Discretization& d, int m, double eta, int far_order, int sing_order, int* nfar,
                      int* nsing) {
  if (m < 2) throw std::invalid_argument("H2Matrix: interpolation degree m < 2");
  if (!(eta > 0)) throw std::invalid_argument("H2Matrix: eta must be positive");
  *nfar = far_order > 0 ? far_order : d.degree() + 2;
  *nsing = sing_order > 0 ? sing_order : d.degree() + 3;
  if (*nfar > 64 || *nsing > 64) throw std::invalid_argument("gauss_rule: order out of range");
}

H2Plan build_plan(const Discretization& d, int m, double eta, int far_order, int sing_order, int partition_device) {
  static const bool verbose = getenv("IGB_VERBOSE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto lap = [&](const char* what) {
    if (!verbose) return;
    const auto now = std::chrono::steady_clock::now();
    fprintf(stderr, "[igb plan] %-14s %8.2f ms\n", what, std::chrono::duration<double, std::milli>(now - tp).count());
    tp = now;
  };
  H2Plan P;
  check_h2_options(d, m, eta, far_order, sing_order, &P.nfar, &P.nsing);
  P.m = m;
  P.eta = eta;
  const int L = d.level(), np = d.geometry().patch_count(), ne = d.element_count();
  P.depth = L;
  P.n_patches = np;
  P.level_offset.resize(L + 1);
  for (int l = 0; l <= L; ++l) {
    P.level_offset[l] = P.npp;
    P.npp += (1 << l) * (1 << l);
  }
  P.n_nodes = np * P.npp;
  const int nn = P.n_nodes;
  P.node_patch.resize(nn);
  P.node_level.resize(nn);
  P.node_sx.resize(nn);
  P.node_sy.resize(nn);
  P.node_box.resize(nn);
  for (int p = 0; p < np; ++p)  // h2.cpp:49-78
    for (int l = L; l >= 0; --l) {
      const int n = 1 << l;
      for (int sy = 0; sy < n; ++sy)
        for (int sx = 0; sx < n; ++sx) {
          const int id = static_cast<int>(P.node_id(p, l, sx, sy));
          P.node_patch[id] = p;
          P.node_level[id] = l;
          P.node_sx[id] = sx;
          P.node_sy[id] = sy;
          if (partition_device >= 0) {
            // boxes come from the device (device_partition)
          } else if (l == L) {
            P.node_box[id] = d.element(d.element_index(p, sx, sy)).box;
          } else {
            Box b;
            b.set_empty();
            for (int k = 0; k < 4; ++k)
              b.extend(P.node_box[P.node_id(p, l + 1, 2 * sx + (k & 1), 2 * sy + (k >> 1))]);
            P.node_box[id] = b;
          }
        }
    }
  lap("tree");
  // dual traversal (h2.cpp:198-216).  Same-level recursion from every ordered
  // root pair; decided pairs of levels 0-1 are collected serially and the
  // undecided level-2 pairs are traversed in parallel (balanced work list).
  std::vector<double> diag(partition_device >= 0 ? 0 : nn);
  if (partition_device >= 0) {
    device_partition(P, d, eta, partition_device);
    lap("device partition");
  } else {
  for (int i = 0; i < nn; ++i) diag[i] = P.node_box[i].diag_norm();
  auto child = [&](int node, int k) {
    return static_cast<int>(P.node_id(P.node_patch[node], P.node_level[node] + 1, 2 * P.node_sx[node] + (k & 1),
                                      2 * P.node_sy[node] + (k >> 1)));
  };
  auto leaf_el = [&](int node) { return d.element_index(P.node_patch[node], P.node_sx[node], P.node_sy[node]); };
  // returns 0 far, 1 near (leaf), 2 recurse
  auto decide = [&](int a, int b) {
    const double dist = P.node_box[a].exterior_distance(P.node_box[b]);
    if (std::max(diag[a], diag[b]) <= eta * dist) return 0;  // h2.cpp:92-97
    return P.node_level[a] == L ? 1 : 2;
  };
  std::vector<std::pair<int, int>> far_top, near_top, work;
  {
    std::vector<std::pair<int, int>> cur;
    for (int pa = 0; pa < np; ++pa)
      for (int pb = 0; pb < np; ++pb)
        cur.emplace_back(static_cast<int>(P.node_id(pa, 0, 0, 0)), static_cast<int>(P.node_id(pb, 0, 0, 0)));
    for (int lev = 0; lev < 2 && !cur.empty(); ++lev) {
      std::vector<std::pair<int, int>> nxt;
      for (auto [a, b] : cur) {
        const int c = decide(a, b);
        if (c == 0) far_top.emplace_back(a, b);
        else if (c == 1) near_top.emplace_back(leaf_el(a), leaf_el(b));
        else
          for (int ka = 0; ka < 4; ++ka)
            for (int kb = 0; kb < 4; ++kb) nxt.emplace_back(child(a, ka), child(b, kb));
      }
      cur.swap(nxt);
    }
    work.swap(cur);
  }
  const int nw = static_cast<int>(work.size());
  std::vector<std::vector<std::pair<int, int>>> far_parts(nw + 1), near_parts(nw + 1);
  far_parts[nw] = std::move(far_top);
  near_parts[nw] = std::move(near_top);
#pragma omp parallel for schedule(dynamic, 4)
  for (int w = 0; w < nw; ++w) {
    auto& fo = far_parts[w];
    auto& no = near_parts[w];
    auto traverse = [&](auto&& self, int a, int b) -> void {
      const int c = decide(a, b);
      if (c == 0) {
        fo.emplace_back(a, b);
        return;
      }
      if (c == 1) {
        no.emplace_back(leaf_el(a), leaf_el(b));
        return;
      }
      for (int ka = 0; ka < 4; ++ka)
        for (int kb = 0; kb < 4; ++kb) self(self, child(a, ka), child(b, kb));
    };
    traverse(traverse, work[w].first, work[w].second);
  }
  lap("traversal");
  // counting sort by row with per-thread histograms (stable, parallel), then
  // each short row by column: the lexicographic order of h2.cpp:215-216 and
  // the CSR row starts of h2.cpp:245-251
  auto bucket = [&](std::vector<std::vector<std::pair<int, int>>>& parts, int nrows, std::vector<int>& A,
                    std::vector<int>& B, std::vector<int>& rs) {
    const int nparts = static_cast<int>(parts.size());
    long long tot = 0;
    for (const auto& v : parts) tot += static_cast<long long>(v.size());
    if (tot > 0x7fffffffLL) throw std::runtime_error("B200 H2: too many block pairs for 32-bit indexing");
    const int T = std::max(1, std::min(omp_get_max_threads(), nparts));
    std::vector<std::vector<int>> hist(T, std::vector<int>(nrows, 0));
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t)
      for (int i = static_cast<int>(static_cast<long long>(nparts) * t / T);
           i < static_cast<int>(static_cast<long long>(nparts) * (t + 1) / T); ++i)
        for (const auto& pr : parts[i]) ++hist[t][pr.first];
    rs.assign(nrows + 1, 0);
    {
      int run = 0;
      for (int r = 0; r < nrows; ++r) {
        rs[r] = run;
        for (int t = 0; t < T; ++t) {
          const int c = hist[t][r];
          hist[t][r] = run;
          run += c;
        }
      }
      rs[nrows] = run;
    }
    B.assign(tot, 0);
    A.resize(tot);
#pragma omp parallel for num_threads(T) schedule(static, 1)
    for (int t = 0; t < T; ++t)
      for (int i = static_cast<int>(static_cast<long long>(nparts) * t / T);
           i < static_cast<int>(static_cast<long long>(nparts) * (t + 1) / T); ++i) {
        for (const auto& pr : parts[i]) B[hist[t][pr.first]++] = pr.second;
        std::vector<std::pair<int, int>>().swap(parts[i]);
      }
#pragma omp parallel for schedule(dynamic, 1024)
    for (int r = 0; r < nrows; ++r) {
      std::sort(B.begin() + rs[r], B.begin() + rs[r + 1]);
      for (int q = rs[r]; q < rs[r + 1]; ++q) A[q] = r;
    }
  };
  bucket(far_parts, nn, P.far_a, P.far_b, P.far_row_start);
  bucket(near_parts, ne, P.near_a, P.near_b, P.near_row_start);
  lap("sort");
  const long long nfar_pairs = static_cast<long long>(P.far_a.size());
  lap("row starts");
  // symmetric structure of the admissible pairs: (t, s) <-> (s, t).  Pairs
  // (s, t) enumerated row-major and bucketed stably by t arrive in (t, s) order,
  // i.e. at the position of their transpose: an O(N) counting sort.
  P.far_trans.assign(nfar_pairs, -1);
  {
    std::vector<int> fillp(P.far_row_start.begin(), P.far_row_start.end() - 1);
    for (long long q = 0; q < nfar_pairs; ++q) P.far_trans[fillp[P.far_b[q]]++] = static_cast<int>(q);
    for (int t = 0; t < nn; ++t)
      if (fillp[t] != P.far_row_start[t + 1]) throw std::logic_error("B200 H2: admissible relation is not symmetric");
  }
  P.far_upper_start.resize(nn);
  int asym = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(+ : asym)
  for (int t = 0; t < nn; ++t) {
    const auto first = P.far_b.begin() + P.far_row_start[t], last = P.far_b.begin() + P.far_row_start[t + 1];
    P.far_upper_start[t] = static_cast<int>(std::upper_bound(first, last, t) - P.far_b.begin());
    for (int q = P.far_row_start[t]; q < P.far_row_start[t + 1]; ++q) {
      const int tq = P.far_trans[q];
      if (P.far_a[tq] != P.far_b[q] || P.far_b[tq] != t) ++asym;
    }
  }
  if (asym) throw std::logic_error("B200 H2: admissible relation is not symmetric");
  lap("transposes");
  }  // host partition
  const long long nnear = static_cast<long long>(P.near_a.size());
  // classification + unique singular work lists
  const bool dev_cls = partition_device >= 0 && static_cast<long long>(P.near_cls.size()) == nnear;
  P.near_cls.resize(nnear);
  std::vector<uint8_t> mapa(nnear), mapb(nnear);
  if (dev_cls) {  // classified on the device
    mapa = P.dev_map_a;
    mapb = P.dev_map_b;
  }
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < (dev_cls ? 0 : nnear); ++q) {
    const int ea = P.near_a[q], eb = P.near_b[q];
    const PairInfo info = d.classify_pair(std::min(ea, eb), std::max(ea, eb));
    P.near_cls[q] = static_cast<uint8_t>(info.cls);
    mapa[q] = static_cast<uint8_t>(info.map_a.bits());
    mapb[q] = static_cast<uint8_t>(info.map_b.bits());
  }
  auto find_slot = [&](int ea, int eb) -> int {
    const auto first = P.near_b.begin() + P.near_row_start[ea];
    const auto last = P.near_b.begin() + P.near_row_start[ea + 1];
    const auto it = std::lower_bound(first, last, eb);
    if (it == last || *it != eb) return -1;
    return static_cast<int>(it - P.near_b.begin());
  };
  // unique singular work items (ea <= eb) per class and the regular slots, in
  // near-list order: per-class prefix sums, then a parallel fill
  std::vector<unsigned char> kind(nnear);  // 0 regular, 1..3 singular item, 4 skip (ea > eb singular)
#pragma omp parallel for schedule(static)
  for (long long q = 0; q < nnear; ++q) {
    const int c = P.near_cls[q];
    kind[q] = c == kFar ? 0 : (P.near_a[q] > P.near_b[q] ? 4 : static_cast<unsigned char>(c));
  }
  std::vector<long long> pos(nnear);
  long long counts[5] = {0, 0, 0, 0, 0};
  for (long long q = 0; q < nnear; ++q) pos[q] = counts[kind[q]]++;
  P.reg_slot.resize(counts[0]);
  for (int c = 1; c <= 3; ++c) {
    auto& L2 = P.sing[c];
    L2.ea.resize(counts[c]);
    L2.eb.resize(counts[c]);
    L2.map_a.resize(counts[c]);
    L2.map_b.resize(counts[c]);
    L2.slot_ab.resize(counts[c]);
    L2.slot_ba.resize(counts[c]);
  }
  int missing = 0;
#pragma omp parallel for schedule(static) reduction(+ : missing)
  for (long long q = 0; q < nnear; ++q) {
    const int k = kind[q];
    if (k == 4) continue;
    if (k == 0) {
      P.reg_slot[pos[q]] = static_cast<int>(q);
      continue;
    }
    const int ea = P.near_a[q], eb = P.near_b[q];
    auto& L2 = P.sing[k];
    const long long i = pos[q];
    L2.ea[i] = ea;
    L2.eb[i] = eb;
    L2.map_a[i] = mapa[q];
    L2.map_b[i] = mapb[q];
    L2.slot_ab[i] = static_cast<int>(q);
    const int sba = ea == eb ? static_cast<int>(q) : find_slot(eb, ea);
    if (sba < 0) ++missing;
    L2.slot_ba[i] = sba;
  }
  if (missing) throw std::logic_error("B200 H2: near relation is not symmetric");
  // unique regular pairs (ea < eb) with both ordered slots: the block of (eb, ea)
  // is the transpose of (ea, eb) (tensor Gauss rule on both elements, symmetric
  // kernel), so the device integrates each pair once
  {
    const long long nreg = static_cast<long long>(P.reg_slot.size());
    std::vector<long long> rpos(nreg + 1, 0);
    for (long long i = 0; i < nreg; ++i) {
      const int q = P.reg_slot[i];
      rpos[i + 1] = rpos[i] + (P.near_a[q] < P.near_b[q] ? 1 : 0);
    }
    P.reg_ab.resize(rpos[nreg]);
    P.reg_ba.resize(rpos[nreg]);
    int miss = 0;
#pragma omp parallel for schedule(static) reduction(+ : miss)
    for (long long i = 0; i < nreg; ++i) {
      const int q = P.reg_slot[i];
      if (P.near_a[q] >= P.near_b[q]) continue;
      const int qb = find_slot(P.near_b[q], P.near_a[q]);
      if (qb < 0) ++miss;
      P.reg_ab[rpos[i]] = q;
      P.reg_ba[rpos[i]] = qb;
    }
    if (miss) throw std::logic_error("B200 H2: near relation is not symmetric");
  }
  lap("classify");
  // DOF incidence in ascending (e, l) order (h2.cpp:359-376 scatter order)
  const int nl = d.local_count(), nd = d.dof_count();
  P.dof_start.assign(nd + 1, 0);
  for (size_t i = 0; i < d.l2g().size(); ++i) ++P.dof_start[d.l2g()[i] + 1];
  for (int i = 0; i < nd; ++i) P.dof_start[i + 1] += P.dof_start[i];
  P.dof_inc.resize(d.l2g().size());
  std::vector<int> fillp(P.dof_start.begin(), P.dof_start.end() - 1);
  for (int e = 0; e < ne; ++e)
    for (int l = 0; l < nl; ++l) {
      const int i = e * nl + l;
      P.dof_inc[fillp[d.l2g()[i]]++] = i;
    }
  lap("dof incidence");
  // interpolation (h2.cpp:113-125)
  P.cheb = cheb_nodes(m);
  P.tl.assign(m * m, 0.0);
  P.tr.assign(m * m, 0.0);
  std::vector<double> ll(m), lr(m);
  for (int j = 0; j < m; ++j) {
    lagrange_all(P.cheb, 0.5 * P.cheb[j], ll.data());
    lagrange_all(P.cheb, 0.5 + 0.5 * P.cheb[j], lr.data());
    for (int i = 0; i < m; ++i) {
      P.tl[i + m * j] = ll[i];
      P.tr[i + m * j] = lr[i];
    }
  }
  return P;
}

int node_cluster(const H2Plan& P, int node) {
  const int l = P.node_level[node];
  if (l == 0) return -1;
  const int sx = P.node_sx[node] >> (l - 1), sy = P.node_sy[node] >> (l - 1);
  return 4 * P.node_patch[node] + sx + 2 * sy;
}

std::vector<unsigned char> owned_elements(const Discretization& d, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("partition: bad rank/world");
  const int ncl = d.level() >= 1 ? 4 * d.geometry().patch_count() : 1;
  const int c0 = static_cast<int>(static_cast<long long>(ncl) * rank / world);
  const int c1 = static_cast<int>(static_cast<long long>(ncl) * (rank + 1) / world);
  const int ne = d.element_count(), n = 1 << d.level();
  std::vector<unsigned char> own(ne, 0);
  for (int e = 0; e < ne; ++e) {
    const Element& el = d.element(e);
    const int cl = d.level() >= 1 ? 4 * el.patch + (el.ix >= n / 2 ? 1 : 0) + 2 * (el.iy >= n / 2 ? 1 : 0) : 0;
    own[e] = cl >= c0 && cl < c1;
  }
  return own;
}

RowPartition partition_rows(const Discretization& d, const H2Plan& P, int world, int rank) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("partition: bad rank/world");
  RowPartition r;
  const int ncl = d.level() >= 1 ? 4 * P.n_patches : 1;
  r.c0 = static_cast<int>(static_cast<long long>(ncl) * rank / world);
  r.c1 = static_cast<int>(static_cast<long long>(ncl) * (rank + 1) / world);
  const int ne = d.element_count();
  r.owns_element = owned_elements(d, world, rank);
  for (int e = 0; e < ne; ++e)
    if (r.owns_element[e]) r.elements.push_back(e);
  for (int e : r.elements) r.near_count += P.near_row_start[e + 1] - P.near_row_start[e];
  for (size_t q = 0; q < P.far_a.size(); ++q) {
    const int cl = node_cluster(P, P.far_a[q]);
    if (cl < 0 || (cl >= r.c0 && cl < r.c1)) ++r.far_count;
  }
  return r;
}

LocalPlan build_local_plan(const Discretization& d, const H2Plan& P, int world, int rank) {
  LocalPlan Lp;
  Lp.world = world;
  Lp.rank = rank;
  const int ne = d.element_count(), nl = d.local_count(), nn = P.n_nodes;
  std::vector<RowPartition> parts;
  for (int r = 0; r < world; ++r) parts.push_back(partition_rows(d, P, world, r));
  const RowPartition& me = parts[rank];
  Lp.c0 = me.c0;
  Lp.c1 = me.c1;
  Lp.el = me.elements;
  Lp.el_local.assign(ne, -1);
  for (size_t i = 0; i < Lp.el.size(); ++i) Lp.el_local[Lp.el[i]] = static_cast<int>(i);
  // near rows
  const long long nnear = static_cast<long long>(P.near_a.size());
  Lp.slot_local.assign(nnear, -1);
  Lp.near_rs.assign(Lp.el.size() + 1, 0);
  for (size_t i = 0; i < Lp.el.size(); ++i) {
    const int e = Lp.el[i];
    Lp.near_rs[i + 1] = Lp.near_rs[i] + (P.near_row_start[e + 1] - P.near_row_start[e]);
    for (int q = P.near_row_start[e]; q < P.near_row_start[e + 1]; ++q) {
      Lp.slot_local[q] = static_cast<int>(Lp.near_row.size());
      Lp.near_row.push_back(static_cast<int>(i));
      Lp.near_ea.push_back(e);
      Lp.near_eb.push_back(P.near_b[q]);
    }
  }
  for (int c = 1; c <= 3; ++c) {
    const auto& G = P.sing[c];
    auto& L = Lp.sing[c];
    for (size_t k = 0; k < G.ea.size(); ++k) {
      const int sab = Lp.slot_local[G.slot_ab[k]], sba = Lp.slot_local[G.slot_ba[k]];
      if (sab < 0 && sba < 0) continue;
      L.ea.push_back(G.ea[k]);
      L.eb.push_back(G.eb[k]);
      L.map_a.push_back(G.map_a[k]);
      L.map_b.push_back(G.map_b[k]);
      L.slot_ab.push_back(sab);
      L.slot_ba.push_back(G.slot_ba[k] == G.slot_ab[k] ? sab : sba);
    }
  }
  for (int q : P.reg_slot)
    if (Lp.slot_local[q] >= 0) Lp.reg_slot.push_back(Lp.slot_local[q]);
  for (size_t i = 0; i < P.reg_ab.size(); ++i) {
    const int a = Lp.slot_local[P.reg_ab[i]], b = Lp.slot_local[P.reg_ba[i]];
    if (a < 0 && b < 0) continue;
    Lp.reg_ab.push_back(a);
    Lp.reg_ba.push_back(b);
  }
  // tree nodes
  Lp.node_owned.assign(nn, 0);
  Lp.rank_pack_nodes.assign(world, {});
  for (int t = 0; t < nn; ++t) {
    const int cl = node_cluster(P, t);
    if (cl < 0) {
      Lp.node_owned[t] = 1;  // roots: replicated on every rank
      continue;
    }
    for (int r = 0; r < world; ++r)
      if (cl >= parts[r].c0 && cl < parts[r].c1) {
        Lp.rank_pack_nodes[r].push_back(t);
        if (r == rank) Lp.node_owned[t] = 1;
      }
  }
  Lp.pack_nodes = Lp.rank_pack_nodes[rank];
  for (const auto& v : Lp.rank_pack_nodes) Lp.pack_max = std::max<int>(Lp.pack_max, static_cast<int>(v.size()));
  for (int t = 0; t < nn; ++t)
    if (Lp.node_owned[t] && P.far_row_start[t + 1] > P.far_row_start[t]) Lp.far_targets.push_back(t);
  // DOF gather over owned elements, ascending (e, l)
  const int nd = d.dof_count();
  Lp.dof_start.assign(nd + 1, 0);
  for (int e : Lp.el)
    for (int l = 0; l < nl; ++l) ++Lp.dof_start[d.l2g()[static_cast<size_t>(e) * nl + l] + 1];
  for (int i = 0; i < nd; ++i) Lp.dof_start[i + 1] += Lp.dof_start[i];
  Lp.dof_inc.resize(Lp.dof_start[nd]);
  std::vector<int> fillp(Lp.dof_start.begin(), Lp.dof_start.end() - 1);
  for (size_t i = 0; i < Lp.el.size(); ++i)
    for (int l = 0; l < nl; ++l) {
      const int e = Lp.el[i];
      Lp.dof_inc[fillp[d.l2g()[static_cast<size_t>(e) * nl + l]]++] = static_cast<int>(i) * nl + l;
    }
  return Lp;
}

}  // namespace igb
