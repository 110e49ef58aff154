// ============================================================================
// oracle/igb_oracle.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A CPU restatement (plain C++17 + OpenMP, no Eigen) of the reference's hot
// path: igabem v0.1.0 under /root/reference/proj/core.  Only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
// may load this library, and only as the checker / the timed CPU baseline.
// The product (paper_1906_00785_b200/) never links or calls it.
//
// Every function cites the reference file:line it restates.  Floating-point
// operation order follows the reference expression by expression wherever the
// result feeds an integer decision (element boxes -> admissibility -> block
// partition), so the partition is bit-identical; elsewhere it follows the
// reference closely (small dense products are plain loops, the only
// difference to the Eigen build is summation order at the 1e-16 level).
//
// Parity pins: the frozen constants of the
// reference's own tests (test_quadrature.cpp:16-18, test_assembly.cpp:53-82),
// the reference test identities re-stated in tests/test_oracle.py, and golden
// vectors produced by the reference itself (oracle/_ref, built against an
// Eigen-subset shim) committed under tests/golden/.
// ============================================================================
#include <algorithm>
#include <array>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace orc {

using cplx = std::complex<double>;

// ---------------------------------------------------------------- vectors
struct V3 {
  double c[3] = {0, 0, 0};
  V3() = default;
  V3(double a, double b, double d) : c{a, b, d} {}
  double& operator[](int i) { return c[i]; }
  double operator[](int i) const { return c[i]; }
};
inline V3 operator+(const V3& a, const V3& b) { return {a[0] + b[0], a[1] + b[1], a[2] + b[2]}; }
inline V3 operator-(const V3& a, const V3& b) { return {a[0] - b[0], a[1] - b[1], a[2] - b[2]}; }
inline V3 operator*(const V3& a, double s) { return {a[0] * s, a[1] * s, a[2] * s}; }
inline V3 operator*(double s, const V3& a) { return {s * a[0], s * a[1], s * a[2]}; }
inline V3 operator/(const V3& a, double s) { return {a[0] / s, a[1] / s, a[2] / s}; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double sqnorm(const V3& a) { return a[0] * a[0] + a[1] * a[1] + a[2] * a[2]; }
inline double norm(const V3& a) { return std::sqrt(sqnorm(a)); }
// Eigen cross product order (Eigen/src/Geometry/OrthoMethods.h)
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}
inline V3 normalized(const V3& a) {
  const double z = sqnorm(a);
  return z > 0 ? a / std::sqrt(z) : a;
}

// Eigen::AlignedBox3d semantics (setEmpty / extend / center / diagonal /
// exteriorDistance), as used by spaces.cpp:133-142 and h2.cpp:69-97.
struct Box {
  double mn[3], mx[3];
  void set_empty() {
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::numeric_limits<double>::max();
      mx[k] = std::numeric_limits<double>::lowest();
    }
  }
  void extend(const V3& p) {
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::min(mn[k], p[k]);
      mx[k] = std::max(mx[k], p[k]);
    }
  }
  void extend(const Box& b) {
    for (int k = 0; k < 3; ++k) {
      mn[k] = std::min(mn[k], b.mn[k]);
      mx[k] = std::max(mx[k], b.mx[k]);
    }
  }
  double diag_norm() const {
    const V3 d(mx[0] - mn[0], mx[1] - mn[1], mx[2] - mn[2]);
    return norm(d);
  }
  double exterior_distance(const Box& b) const {
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
  bool contains(const Box& b) const {
    for (int k = 0; k < 3; ++k)
      if (b.mn[k] < mn[k] || b.mx[k] > mx[k]) return false;
    return true;
  }
};

// ------------------------------------------------------------ quadrature
// quadrature.cpp:15-50
struct Rule1D {
  std::vector<double> nodes, weights;
};
static Rule1D build_gauss(int n) {
  Rule1D r;
  r.nodes.resize(n);
  r.weights.resize(n);
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
    r.nodes[n - 1 - i] = 0.5 * (1.0 + x);
    r.weights[n - 1 - i] = 1.0 / ((1.0 - x * x) * dp * dp);
  }
  return r;
}
static std::mutex g_gauss_mu, g_pair_mu;
const Rule1D& gauss_rule(int n) {
  if (n < 1 || n > 64) throw std::invalid_argument("gauss_rule: order out of range");
  static std::map<int, Rule1D> cache;
  std::lock_guard<std::mutex> lk(g_gauss_mu);
  auto it = cache.find(n);
  if (it == cache.end()) it = cache.emplace(n, build_gauss(n)).first;
  return it->second;
}

enum PairClass { kFar = 0, kVertex = 1, kEdge = 2, kCoincident = 3 };  // quadrature.hpp:17

// quadrature.hpp:22-30
struct SquareMap {
  bool swap = false, flip_u = false, flip_v = false;
  void apply(double& u, double& v) const {
    if (swap) std::swap(u, v);
    if (flip_u) u = 1.0 - u;
    if (flip_v) v = 1.0 - v;
  }
};
// quadrature.cpp:52-63
SquareMap map_bottom_to_edge(int edge, bool reversed) {
  switch (edge) {
    case 0: return {false, reversed, false};
    case 1: return {true, true, reversed};
    case 2: return {false, reversed, true};
    case 3: return {true, false, reversed};
  }
  throw std::logic_error("map_bottom_to_edge: bad edge");
}
// quadrature.cpp:65-73
SquareMap map_origin_to_corner(int corner) {
  switch (corner) {
    case 0: return {false, false, false};
    case 1: return {false, true, false};
    case 2: return {false, false, true};
    case 3: return {false, true, true};
  }
  throw std::logic_error("map_origin_to_corner: bad corner");
}

struct PairPoint {
  double ua, va, ub, vb, w;
};
// quadrature.cpp:82-111
static std::vector<PairPoint> build_coincident(int n) {
  const auto& g = gauss_rule(n);
  std::vector<PairPoint> pts;
  pts.reserve(8 * n * n * n * n);
  for (int axis = 0; axis < 2; ++axis)
    for (int dir : {1, -1})
      for (int sgn : {1, -1})
        for (int i1 = 0; i1 < n; ++i1)
          for (int i2 = 0; i2 < n; ++i2)
            for (int i3 = 0; i3 < n; ++i3)
              for (int i4 = 0; i4 < n; ++i4) {
                const double t = g.nodes[i1], s = g.nodes[i2];
                double z1, z2;
                if (axis == 0) {
                  z1 = dir * t;
                  z2 = sgn * t * s;
                } else {
                  z1 = sgn * t * s;
                  z2 = dir * t;
                }
                const double lx = 1.0 - std::abs(z1), ly = 1.0 - std::abs(z2);
                const double x1 = std::max(0.0, -z1) + lx * g.nodes[i3];
                const double x2 = std::max(0.0, -z2) + ly * g.nodes[i4];
                const double w = g.weights[i1] * g.weights[i2] * g.weights[i3] *
                                 g.weights[i4] * t * lx * ly;
                pts.push_back({x1, x2, x1 + z1, x2 + z2, w});
              }
  return pts;
}
// quadrature.cpp:113-149
static std::vector<PairPoint> build_edge(int n) {
  const auto& g = gauss_rule(n);
  std::vector<PairPoint> pts;
  pts.reserve(6 * n * n * n * n);
  auto emit = [&](int kind, int sgn) {
    for (int i1 = 0; i1 < n; ++i1)
      for (int i2 = 0; i2 < n; ++i2)
        for (int i3 = 0; i3 < n; ++i3)
          for (int i4 = 0; i4 < n; ++i4) {
            const double t = g.nodes[i1], a = g.nodes[i2], b = g.nodes[i3];
            double d, va, vb, jac;
            switch (kind) {
              case 0:
                va = t; vb = t * b; d = sgn * t * a;
                jac = t * t * (1.0 - t * a);
                break;
              case 1:
                vb = t; va = t * b; d = sgn * t * a;
                jac = t * t * (1.0 - t * a);
                break;
              default:
                d = sgn * t; va = t * a; vb = t * b;
                jac = t * t * (1.0 - t);
                break;
            }
            const double ua = std::max(0.0, -d) + (1.0 - std::abs(d)) * g.nodes[i4];
            const double w =
                g.weights[i1] * g.weights[i2] * g.weights[i3] * g.weights[i4] * jac;
            pts.push_back({ua, va, ua + d, vb, w});
          }
  };
  for (int kind = 0; kind < 3; ++kind)
    for (int sgn : {1, -1}) emit(kind, sgn);
  return pts;
}
// quadrature.cpp:151-177
static std::vector<PairPoint> build_vertex(int n) {
  const auto& g = gauss_rule(n);
  std::vector<PairPoint> pts;
  pts.reserve(4 * n * n * n * n);
  for (int dom = 0; dom < 4; ++dom)
    for (int i1 = 0; i1 < n; ++i1)
      for (int i2 = 0; i2 < n; ++i2)
        for (int i3 = 0; i3 < n; ++i3)
          for (int i4 = 0; i4 < n; ++i4) {
            const double t = g.nodes[i1];
            double c[4];
            int j = 0;
            const double vals[3] = {g.nodes[i2], g.nodes[i3], g.nodes[i4]};
            for (int k = 0; k < 4; ++k) c[k] = (k == dom) ? t : t * vals[j++];
            const double w = g.weights[i1] * g.weights[i2] * g.weights[i3] *
                             g.weights[i4] * t * t * t;
            pts.push_back({c[0], c[1], c[2], c[3], w});
          }
  return pts;
}
// quadrature.cpp:181-199
const std::vector<PairPoint>& pair_rule(int cls, int n) {
  if (cls == kFar) throw std::logic_error("pair_rule: Far pairs use tensor Gauss directly");
  static std::map<std::pair<int, int>, std::vector<PairPoint>> cache;
  gauss_rule(n);  // validates n, outside the pair lock
  std::lock_guard<std::mutex> lk(g_pair_mu);
  const auto key = std::make_pair(cls, n);
  auto it = cache.find(key);
  if (it == cache.end()) {
    std::vector<PairPoint> pts;
    if (cls == kVertex) pts = build_vertex(n);
    if (cls == kEdge) pts = build_edge(n);
    if (cls == kCoincident) pts = build_coincident(n);
    it = cache.emplace(key, std::move(pts)).first;
  }
  return it->second;
}

// --------------------------------------------------------------- splines
// splines.hpp:11-31, splines.cpp:7-52
struct KnotVector {
  std::vector<double> knots;
  int degree = 0;
  int size() const { return static_cast<int>(knots.size()) - degree - 1; }
  int find_span(double x) const {  // splines.cpp:20-38
    const int p = degree;
    const int k = size();
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
};
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

// splines.cpp:69-86 (local de Boor triangle); out has p+1 entries
static void basis_values(const KnotVector& kv, int span, double x, double* out) {
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
// splines.cpp:122-171 (derivatives as expanded differences)
static void deriv_values(const KnotVector& kv, int span, double x, int order, double* out) {
  if (order != 1 && order != 2)
    throw std::invalid_argument("eval_basis_deriv: order must be 1 or 2");
  const int p = kv.degree;
  for (int i = 0; i <= p; ++i) out[i] = 0.0;
  if (order > p) return;
  const int q = p - order;
  double low[32];
  {
    KnotVector sub = kv;
    sub.degree = q;
    basis_values(sub, span, x, low);
  }
  const int first = span - p;
  for (int i = 0; i <= p; ++i) {
    std::vector<double> c(1, 1.0);
    int lo = first + i;
    int deg = p;
    for (int m = 0; m < order; ++m) {
      std::vector<double> nc(c.size() + 1, 0.0);
      for (size_t r = 0; r < c.size(); ++r) {
        const int j = lo + static_cast<int>(r);
        const double d1 = kv.knots[j + deg] - kv.knots[j];
        const double d2 = kv.knots[j + deg + 1] - kv.knots[j + 1];
        if (d1 > 0.0) nc[r] += c[r] * deg / d1;
        if (d2 > 0.0) nc[r + 1] -= c[r] * deg / d2;
      }
      c = std::move(nc);
      --deg;
    }
    double v = 0.0;
    for (size_t r = 0; r < c.size(); ++r) {
      const int j = lo + static_cast<int>(r);
      const int off = j - (span - q);
      if (off >= 0 && off <= q) v += c[r] * low[off];
    }
    out[i] = v;
  }
}
static void check_domain(double x) {
  if (!(x >= 0.0 && x <= 1.0)) throw std::domain_error("eval_basis: parameter outside [0,1]");
}
int eval_basis(const KnotVector& kv, double x, double* out) {  // splines.cpp:88-93
  check_domain(x);
  const int span = kv.find_span(x);
  basis_values(kv, span, x, out);
  return span - kv.degree;
}
int eval_basis_deriv(const KnotVector& kv, double x, int order, double* out) {
  check_domain(x);
  const int span = kv.find_span(x);
  deriv_values(kv, span, x, order, out);
  return span - kv.degree;
}

// splines.hpp:53-67: homogeneous control points ctrl_w (3 x n) and weights
struct Patch {
  KnotVector kv_u, kv_v;
  std::vector<double> cw;  // 3 * n, column i + j*ku
  std::vector<double> w;   // n
  int count_u() const { return kv_u.size(); }
  int count_v() const { return kv_v.size(); }
  V3 point(int i, int j) const {
    const int idx = i + j * count_u();
    return V3(cw[3 * idx], cw[3 * idx + 1], cw[3 * idx + 2]) / w[idx];
  }
  void validate() const {  // splines.cpp:206-211
    const int n = count_u() * count_v();
    if (static_cast<int>(w.size()) != n || static_cast<int>(cw.size()) != 3 * n)
      throw std::invalid_argument("PatchSurface: control grid does not match basis counts");
    for (double x : w)
      if (x <= 0.0) throw std::invalid_argument("PatchSurface: weights must be strictly positive");
  }
};
struct Jet {
  V3 x, du, dv;
};
// splines.cpp:183-216
Jet eval_patch(const Patch& s, double u, double v) {
  double bu[32], bv[32], du[32], dv[32];
  const int fu = eval_basis(s.kv_u, u, bu);
  const int fv = eval_basis(s.kv_v, v, bv);
  eval_basis_deriv(s.kv_u, u, 1, du);
  eval_basis_deriv(s.kv_v, v, 1, dv);
  const int pu = s.kv_u.degree, pv = s.kv_v.degree;
  const int ku = s.count_u();
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

// -------------------------------------------------------------- geometry
struct EdgeIdent {
  int patch_a, edge_a, patch_b, edge_b;
  bool reversed;
};
struct VertexIdent {
  int patch_a, corner_a, patch_b, corner_b;
};
struct Frame {
  V3 x, du, dv, normal;
  double sqrt_g;
};
void edge_point(int edge, double t, double& u, double& v) {  // geometry.cpp:72-80
  switch (edge) {
    case 0: u = t; v = 0; break;
    case 1: u = 1; v = t; break;
    case 2: u = t; v = 1; break;
    case 3: u = 0; v = t; break;
    default: throw std::logic_error("edge_point: bad edge");
  }
}

struct Geometry {
  std::vector<Patch> patches;
  std::vector<EdgeIdent> edges;
  std::vector<VertexIdent> vertices;

  int patch_count() const { return static_cast<int>(patches.size()); }
  Frame frame(int p, double u, double v) const {  // geometry.cpp:167-176
    const Jet j = eval_patch(patches[p], u, v);
    Frame f;
    f.x = j.x;
    f.du = j.du;
    f.dv = j.dv;
    f.normal = cross(j.du, j.dv);
    f.sqrt_g = norm(f.normal);
    return f;
  }
  std::vector<V3> edge_polygon(const Patch& s, int edge) const {  // geometry.cpp:17-45
    const int ku = s.count_u(), kv = s.count_v();
    std::vector<V3> poly;
    switch (edge) {
      case 0: for (int i = 0; i < ku; ++i) poly.push_back(s.point(i, 0)); break;
      case 1: for (int j = 0; j < kv; ++j) poly.push_back(s.point(ku - 1, j)); break;
      case 2: for (int i = 0; i < ku; ++i) poly.push_back(s.point(i, kv - 1)); break;
      case 3: for (int j = 0; j < kv; ++j) poly.push_back(s.point(0, j)); break;
    }
    return poly;
  }
  static bool polys_match(const std::vector<V3>& a, const std::vector<V3>& b, bool& rev) {
    if (a.size() != b.size()) return false;  // geometry.cpp:53-70
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
  V3 corner_ctrl(const Patch& s, int corner) const {
    const int i = (corner == 1 || corner == 3) ? s.count_u() - 1 : 0;
    const int j = (corner >= 2) ? s.count_v() - 1 : 0;
    return s.point(i, j);
  }
  void infer_topology() {  // geometry.cpp:96-124
    const int m = patch_count();
    std::vector<int> paired(4 * m, 0);
    for (int a = 0; a < m; ++a)
      for (int ea = 0; ea < 4; ++ea) {
        const auto pa = edge_polygon(patches[a], ea);
        for (int b = a; b < m; ++b)
          for (int eb = (b == a ? ea + 1 : 0); eb < 4; ++eb) {
            bool rev = false;
            if (polys_match(pa, edge_polygon(patches[b], eb), rev)) {
              edges.push_back({a, ea, b, eb, rev});
              if (++paired[4 * a + ea] > 1 || ++paired[4 * b + eb] > 1)
                throw std::runtime_error("Geometry: three or more coincident edges");
            }
          }
      }
    for (int a = 0; a < m; ++a)
      for (int ca = 0; ca < 4; ++ca) {
        const V3 xa = corner_ctrl(patches[a], ca);
        for (int b = a; b < m; ++b)
          for (int cb = (b == a ? ca + 1 : 0); cb < 4; ++cb)
            if (norm(xa - corner_ctrl(patches[b], cb)) <= 1e-9) vertices.push_back({a, ca, b, cb});
      }
  }
  void validate_regularity() const {  // geometry.cpp:126-139
    for (int p = 0; p < patch_count(); ++p)
      for (int i = 0; i < 5; ++i)
        for (int j = 0; j < 5; ++j)
          if (frame(p, i / 4.0, j / 4.0).sqrt_g < 1e-12)
            throw std::runtime_error("Geometry: degenerate parametrization");
  }
  bool is_closed() const { return static_cast<int>(edges.size()) == 2 * patch_count(); }
  void validate_orientation() const {  // geometry.cpp:141-163
    if (!is_closed()) return;
    V3 centroid;
    int n = 0;
    for (int p = 0; p < patch_count(); ++p)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          centroid = centroid + frame(p, 0.25 + 0.25 * i, 0.25 + 0.25 * j).x;
          ++n;
        }
    centroid = centroid / n;
    for (int p = 0; p < patch_count(); ++p)
      for (int i = 0; i < 3; ++i)
        for (int j = 0; j < 3; ++j) {
          const Frame f = frame(p, 0.25 + 0.25 * i, 0.25 + 0.25 * j);
          if (dot(f.normal, f.x - centroid) <= 0.0)
            throw std::runtime_error("Geometry: normal is not outward pointing");
        }
  }
  double check_matching() const {  // geometry.cpp:178-195; returns max deviation
    double worst = 0;
    for (const auto& e : edges) {
      double dev = 0;
      for (int k = 0; k < 17; ++k) {
        const double t = k / 16.0;
        const double tb = e.reversed ? 1.0 - t : t;
        double ua, va, ub, vb;
        edge_point(e.edge_a, t, ua, va);
        edge_point(e.edge_b, tb, ub, vb);
        dev = std::max(dev, norm(eval_patch(patches[e.patch_a], ua, va).x -
                                 eval_patch(patches[e.patch_b], ub, vb).x));
      }
      if (dev > 1e-9) worst = std::max(worst, dev);
    }
    return worst;
  }
  void finish() {  // geometry.cpp:88-94
    if (patches.empty()) throw std::invalid_argument("Geometry: no patches");
    for (const auto& p : patches) p.validate();
    infer_topology();
    validate_regularity();
    validate_orientation();
  }
};

// ----------------------------------------------------------------- shapes
// shapes.cpp:9-26
Patch make_rectangle_patch(const V3& origin, const V3& su, const V3& sv, int p) {
  Patch s;
  s.kv_u = make_uniform_knots(p, 0, 1);
  s.kv_v = make_uniform_knots(p, 0, 1);
  const int k = p + 1;
  s.cw.resize(3 * k * k);
  s.w.assign(k * k, 1.0);
  for (int j = 0; j < k; ++j)
    for (int i = 0; i < k; ++i) {
      const double gu = p > 0 ? double(i) / p : 0.5;
      const double gv = p > 0 ? double(j) / p : 0.5;
      const V3 x = origin + su * gu + sv * gv;
      for (int c = 0; c < 3; ++c) s.cw[3 * (i + j * k) + c] = x[c];
    }
  return s;
}
Geometry make_square() {  // shapes.cpp:28-30
  Geometry g;
  g.patches.push_back(make_rectangle_patch({0, 0, 0}, {1, 0, 0}, {0, 1, 0}, 1));
  g.finish();
  return g;
}

// bivariate power-basis polynomial coef(i,j) u^i v^j (shapes.cpp:34-58)
struct Poly2 {
  int r = 1, c = 1;
  std::vector<double> a;  // column-major
  Poly2() : a(1, 0.0) {}
  Poly2(int rr, int cc) : r(rr), c(cc), a(rr * cc, 0.0) {}
  double& operator()(int i, int j) { return a[i + r * j]; }
  double operator()(int i, int j) const { return a[i + r * j]; }
};
static Poly2 pscale(const Poly2& x, double s) {
  Poly2 y = x;
  for (auto& v : y.a) v = v * s;
  return y;
}
static Poly2 pneg(const Poly2& x) {
  Poly2 y = x;
  for (auto& v : y.a) v = -v;
  return y;
}
static Poly2 pmul(const Poly2& a, const Poly2& b) {
  Poly2 c(a.r + b.r - 1, a.c + b.c - 1);
  for (int i = 0; i < a.r; ++i)
    for (int j = 0; j < a.c; ++j)
      for (int k = 0; k < b.r; ++k)
        for (int l = 0; l < b.c; ++l) c(i + k, j + l) += a(i, j) * b(k, l);
  return c;
}
static Poly2 padd(const Poly2& a, const Poly2& b) {
  Poly2 c(std::max(a.r, b.r), std::max(a.c, b.c));
  for (int j = 0; j < a.c; ++j)
    for (int i = 0; i < a.r; ++i) c(i, j) = a(i, j);
  for (int j = 0; j < b.c; ++j)
    for (int i = 0; i < b.r; ++i) c(i, j) += b(i, j);
  return c;
}
static double binom(int n, int k) {
  double r = 1;
  for (int i = 0; i < k; ++i) r = r * (n - i) / (i + 1);
  return r;
}
static std::vector<double> power_to_bernstein(const std::vector<double>& a, int n) {
  std::vector<double> c(n + 1, 0.0);
  for (int j = 0; j <= n; ++j)
    for (int k = 0; k <= j && k < static_cast<int>(a.size()); ++k)
      c[j] += a[k] * binom(j, k) / binom(n, k);
  return c;
}
struct V4 {
  double c[4];
};
static std::array<V4, 3> arc_h(const V3& A, const V3& B) {  // shapes.cpp:78-85
  const double c = dot(A, B);
  const double w = std::sqrt((1.0 + c) / 2.0);
  const V3 M = (A + B) / (1.0 + c);
  return {V4{{A[0], A[1], A[2], 1.0}}, V4{{w * M[0], w * M[1], w * M[2], w}},
          V4{{B[0], B[1], B[2], 1.0}}};
}
// shapes.cpp:87-205
Geometry make_sphere(double radius, const V3& center) {
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
  Geometry geo;
  for (const auto& face : faces) {
    const V3 a = face.a;
    const V3 ref = std::abs(a[0]) < 0.9 ? V3(1, 0, 0) : V3(0, 1, 0);
    const V3 e1 = normalized(cross(a, ref));
    const V3 e2 = cross(a, e1);
    V3 C[4];
    for (int i = 0; i < 4; ++i) C[i] = face.c[i] * s;
    auto project = [&](const V4& h) {
      const V3 x(h.c[0], h.c[1], h.c[2]);
      return V3(dot(e1, x), dot(e2, x), h.c[3] + dot(a, x));
    };
    auto arc2d = [&](const V3& A, const V3& B) {
      const auto h = arc_h(A, B);
      return std::array<V3, 3>{project(h[0]), project(h[1]), project(h[2])};
    };
    const auto bottom = arc2d(C[0], C[1]);
    const auto top = arc2d(C[2], C[3]);
    const auto left = arc2d(C[0], C[2]);
    const auto right = arc2d(C[1], C[3]);

    Poly2 one(1, 1);
    one(0, 0) = 1.0;
    Poly2 u(2, 1), v(1, 2);
    u(0, 0) = 0; u(1, 0) = 1;
    v(0, 0) = 0; v(0, 1) = 1;
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
      const V3 P00 = bottom[0], P10 = bottom[2], P01 = top[0], P11 = top[2];
      acc = padd(acc, pscale(pmul(mu, mv), -P00[c]));
      acc = padd(acc, pscale(pmul(u, mv), -P10[c]));
      acc = padd(acc, pscale(pmul(mu, v), -P01[c]));
      acc = padd(acc, pscale(pmul(u, v), -P11[c]));
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
      double tmp[5][5];
      for (int j = 0; j < 5; ++j) {
        std::vector<double> col(5);
        for (int i = 0; i < 5; ++i) col[i] = full[i][j];
        const auto b = power_to_bernstein(col, 4);
        for (int i = 0; i < 5; ++i) tmp[i][j] = b[i];
      }
      for (int i = 0; i < 5; ++i) {
        std::vector<double> row(5);
        for (int j = 0; j < 5; ++j) row[j] = tmp[i][j];
        const auto b = power_to_bernstein(row, 4);
        for (int j = 0; j < 5; ++j) full[i][j] = b[j];
      }
      for (int j = 0; j < 5; ++j)
        for (int i = 0; i < 5; ++i) net[c][i + 5 * j] = full[i][j];
    }
    patch.w.resize(25);
    patch.cw.resize(75);
    for (int i = 0; i < 25; ++i) {
      patch.w[i] = net[3][i];
      if (patch.w[i] <= 0.0) throw std::logic_error("make_sphere: nonpositive weight");
    }
    for (int i = 0; i < 25; ++i)
      for (int c = 0; c < 3; ++c) patch.cw[3 * i + c] = radius * net[c][i] + center[c] * net[3][i];
    geo.patches.push_back(std::move(patch));
  }
  geo.finish();
  return geo;
}

// ------------------------------------------------------------ discretization
enum Kind { kLaplace = 0, kHelmholtz = 1, kMaxwell = 2 };  // pde.hpp:9-27

struct Element {  // spaces.hpp:15-21
  int patch, ix, iy;
  double h, ox, oy;
  Box box;
};
struct PairInfo {  // spaces.hpp:32-35
  int cls = kFar;
  SquareMap map_a, map_b;
};
constexpr int kMaxLocal = 64;
struct Shapes {
  int nl = 0;
  double value[kMaxLocal];
  double field[3][kMaxLocal];
  double div[kMaxLocal];
};

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
static bool element_on_edge(int edge, int ix, int iy, int n) {  // spaces.cpp:44-52
  switch (edge) {
    case 0: return iy == 0;
    case 1: return ix == n - 1;
    case 2: return iy == n - 1;
    case 3: return ix == 0;
  }
  return false;
}
static int grid_pos_on_edge(int edge, int ix, int iy) { return (edge == 0 || edge == 2) ? ix : iy; }
static int edge_end_corner(int edge, int end) {
  static const int tbl[4][2] = {{0, 1}, {1, 3}, {2, 3}, {0, 2}};
  return tbl[edge][end];
}
static bool element_at_corner(int corner, int ix, int iy, int n) {
  const int cx = (corner == 1 || corner == 3) ? n - 1 : 0;
  const int cy = (corner >= 2) ? n - 1 : 0;
  return ix == cx && iy == cy;
}

struct Disc {
  std::shared_ptr<Geometry> geom;
  int kind = kLaplace;
  cplx kappa{0, 0};
  int degree = 0, rep = 1, level = 0;
  int epp = 0, n_dofs = 0, n_local = 0;
  KnotVector scalar_kv, vec_kv_p, vec_kv_q;
  int scalar_k = 0, vec_kp = 0, vec_kq = 0;
  std::vector<Element> elements;
  std::vector<int> l2g;       // ne * nl
  std::vector<double> lsign;  // ne * nl
  struct CrossEdge {
    int edge_a, edge_b;
    bool reversed;
  };
  struct CrossCorner {
    int corner_a, corner_b;
  };
  std::vector<std::vector<std::vector<CrossEdge>>> cross_edges;
  std::vector<std::vector<std::vector<CrossCorner>>> cross_corners;

  bool is_complex() const { return kind != kLaplace; }
  bool is_vector() const { return kind == kMaxwell; }
  int ne() const { return static_cast<int>(elements.size()); }
  int element_index(int p, int ix, int iy) const { return p * epp + ix + (1 << level) * iy; }

  // spaces.cpp:71-115
  Disc(std::shared_ptr<Geometry> g, int kind_, cplx kap, int P, int rep_, int L)
      : geom(std::move(g)), kind(kind_), kappa(kap), degree(P), rep(rep_), level(L) {
    if (kind == kMaxwell && kappa == cplx(0, 0))
      throw std::invalid_argument("Pde: Maxwell requires a nonzero wavenumber");
    if (L < 0) throw std::invalid_argument("Discretization: negative level");
    if (kind == kMaxwell) {
      if (P < 1) throw std::invalid_argument("Discretization: Maxwell requires degree P >= 1");
      if (rep != 1)
        throw std::invalid_argument("Discretization: the div-conforming space supports knot repetition 1 only");
    } else if (P < 0) {
      throw std::invalid_argument("Discretization: negative degree");
    }
    if (rep < 1 || rep > std::max(P, 0) + 1)
      throw std::invalid_argument("Discretization: knot repetition out of range");
    if (geom->check_matching() > 0)
      throw std::runtime_error("Discretization: geometry fails the matching condition");
    const int m = geom->patch_count();
    cross_edges.assign(m, std::vector<std::vector<CrossEdge>>(m));
    cross_corners.assign(m, std::vector<std::vector<CrossCorner>>(m));
    for (const auto& e : geom->edges) {
      cross_edges[e.patch_a][e.patch_b].push_back({e.edge_a, e.edge_b, e.reversed});
      cross_edges[e.patch_b][e.patch_a].push_back({e.edge_b, e.edge_a, e.reversed});
    }
    for (const auto& v : geom->vertices) {
      cross_corners[v.patch_a][v.patch_b].push_back({v.corner_a, v.corner_b});
      cross_corners[v.patch_b][v.patch_a].push_back({v.corner_b, v.corner_a});
    }
    build_elements();
    if (kind == kMaxwell)
      build_maxwell();
    else
      build_scalar();
  }

  void build_elements() {  // spaces.cpp:117-147
    const int n = 1 << level;
    const double h = 1.0 / n;
    const int m = geom->patch_count();
    epp = n * n;
    elements.resize(static_cast<size_t>(m) * epp);
    const int ns = degree + 2;
#pragma omp parallel for schedule(static)
    for (int idx = 0; idx < m * epp; ++idx) {
      const int p = idx / epp, r = idx % epp, iy = r / n, ix = r % n;
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
          el.box.extend(eval_patch(geom->patches[p], u, v).x);
        }
      V3 c, half;
      for (int k = 0; k < 3; ++k) c[k] = (el.box.mn[k] + el.box.mx[k]) / 2.0;
      for (int k = 0; k < 3; ++k) half[k] = 1.1 * (el.box.mx[k] - c[k]);
      for (int k = 0; k < 3; ++k) {
        el.box.mn[k] = c[k] - half[k];
        el.box.mx[k] = c[k] + half[k];
      }
      elements[idx] = el;
    }
  }

  void build_scalar() {  // spaces.cpp:149-176
    if (degree == 0)
      scalar_kv = make_uniform_knots(0, level, 1);
    else
      scalar_kv = make_uniform_knots(degree - 1, level, std::min(rep, degree));
    scalar_k = scalar_kv.size();
    const int q = scalar_kv.degree;
    n_local = (q + 1) * (q + 1);
    const int per_patch = scalar_k * scalar_k;
    n_dofs = geom->patch_count() * per_patch;
    l2g.resize(static_cast<size_t>(ne()) * n_local);
    lsign.assign(static_cast<size_t>(ne()) * n_local, 1.0);
    for (int e = 0; e < ne(); ++e) {
      const auto& el = elements[e];
      const double mid = el.ox + 0.5 * el.h;
      const double midv = el.oy + 0.5 * el.h;
      const int fu = scalar_kv.find_span(mid) - q;
      const int fv = scalar_kv.find_span(midv) - q;
      int l = 0;
      for (int j = 0; j <= q; ++j)
        for (int i = 0; i <= q; ++i, ++l)
          l2g[static_cast<size_t>(e) * n_local + l] = el.patch * per_patch + (fu + i) + scalar_k * (fv + j);
    }
  }

  void build_maxwell() {  // spaces.cpp:178-255
    const int P = degree;
    vec_kv_p = make_uniform_knots(P, level, 1);
    vec_kv_q = make_uniform_knots(P - 1, level, 1);
    vec_kp = vec_kv_p.size();
    vec_kq = vec_kv_q.size();
    const int m = geom->patch_count();
    const int per_block = vec_kp * vec_kq;
    const int per_patch = 2 * per_block;
    const int n_raw = m * per_patch;
    auto raw_u = [&](int patch, int i, int j) { return patch * per_patch + i + vec_kp * j; };
    auto raw_v = [&](int patch, int i, int j) { return patch * per_patch + per_block + i + vec_kq * j; };
    auto strip = [&](int patch, int edge, int s) -> std::pair<int, double> {
      switch (edge) {
        case 0: return {raw_v(patch, s, 0), -1.0};
        case 1: return {raw_u(patch, vec_kp - 1, s), +1.0};
        case 2: return {raw_v(patch, s, vec_kp - 1), +1.0};
        case 3: return {raw_u(patch, 0, s), -1.0};
      }
      throw std::logic_error("strip: bad edge");
    };
    SignedUnionFind uf(n_raw);
    for (const auto& e : geom->edges)
      for (int s = 0; s < vec_kq; ++s) {
        const int sb = e.reversed ? vec_kq - 1 - s : s;
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
    n_dofs = next;
    n_local = 2 * (P + 1) * P;
    l2g.resize(static_cast<size_t>(ne()) * n_local);
    lsign.resize(static_cast<size_t>(ne()) * n_local);
    for (int e = 0; e < ne(); ++e) {
      const auto& el = elements[e];
      const double midu = el.ox + 0.5 * el.h;
      const double midv = el.oy + 0.5 * el.h;
      const int fpu = vec_kv_p.find_span(midu) - P;
      const int fpv = vec_kv_p.find_span(midv) - P;
      const int fqu = vec_kv_q.find_span(midu) - (P - 1);
      const int fqv = vec_kv_q.find_span(midv) - (P - 1);
      int l = 0;
      for (int j = 0; j < P; ++j)
        for (int i = 0; i <= P; ++i, ++l) {
          const int r = raw_u(el.patch, fpu + i, fqv + j);
          l2g[static_cast<size_t>(e) * n_local + l] = glob[r];
          lsign[static_cast<size_t>(e) * n_local + l] = gsign[r];
        }
      for (int j = 0; j <= P; ++j)
        for (int i = 0; i < P; ++i, ++l) {
          const int r = raw_v(el.patch, fqu + i, fpv + j);
          l2g[static_cast<size_t>(e) * n_local + l] = glob[r];
          lsign[static_cast<size_t>(e) * n_local + l] = gsign[r];
        }
    }
  }

  // spaces.cpp:257-307
  void sample_shapes(int e, double u_loc, double v_loc, Shapes& out) const {
    const auto& el = elements[e];
    const double u = el.ox + el.h * u_loc;
    const double v = el.oy + el.h * v_loc;
    out.nl = n_local;
    if (!is_vector()) {
      const int q = scalar_kv.degree;
      const int su = scalar_kv.find_span(el.ox + 0.5 * el.h);
      const int sv = scalar_kv.find_span(el.oy + 0.5 * el.h);
      double bu[32], bv[32];
      basis_values(scalar_kv, su, u, bu);
      basis_values(scalar_kv, sv, v, bv);
      for (int j = 0; j <= q; ++j)
        for (int i = 0; i <= q; ++i) out.value[i + (q + 1) * j] = bu[i] * bv[j];
      return;
    }
    const int P = degree;
    const Frame f = geom->frame(el.patch, u, v);
    const double inv_g = 1.0 / f.sqrt_g;
    const int spu = vec_kv_p.find_span(el.ox + 0.5 * el.h);
    const int spv = vec_kv_p.find_span(el.oy + 0.5 * el.h);
    const int squ = vec_kv_q.find_span(el.ox + 0.5 * el.h);
    const int sqv = vec_kv_q.find_span(el.oy + 0.5 * el.h);
    double bpu[32], bpv[32], bqu[32], bqv[32], dpu[32], dpv[32];
    basis_values(vec_kv_p, spu, u, bpu);
    basis_values(vec_kv_p, spv, v, bpv);
    basis_values(vec_kv_q, squ, u, bqu);
    basis_values(vec_kv_q, sqv, v, bqv);
    deriv_values(vec_kv_p, spu, u, 1, dpu);
    deriv_values(vec_kv_p, spv, v, 1, dpv);
    int l = 0;
    for (int j = 0; j < P; ++j)
      for (int i = 0; i <= P; ++i, ++l) {
        const V3 fl = inv_g * f.du * (bpu[i] * bqv[j]);
        for (int d = 0; d < 3; ++d) out.field[d][l] = fl[d];
        out.div[l] = inv_g * dpu[i] * bqv[j];
      }
    for (int j = 0; j <= P; ++j)
      for (int i = 0; i < P; ++i, ++l) {
        const V3 fl = inv_g * f.dv * (bqu[i] * bpv[j]);
        for (int d = 0; d < 3; ++d) out.field[d][l] = fl[d];
        out.div[l] = inv_g * bqu[i] * dpv[j];
      }
  }

  // spaces.cpp:309-394
  PairInfo classify_pair(int ea, int eb) const {
    PairInfo info;
    if (ea == eb) {
      info.cls = kCoincident;
      return info;
    }
    const auto& a = elements[ea];
    const auto& b = elements[eb];
    const int n = 1 << level;
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
      for (const auto& ce : cross_edges[a.patch][b.patch]) {
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
          const int ca = edge_end_corner(ce.edge_a, end_a);
          const int cb = edge_end_corner(ce.edge_b, end_b_pos);
          cand.cls = kVertex;
          cand.map_a = map_origin_to_corner(ca);
          cand.map_b = map_origin_to_corner(cb);
          best = 1;
        }
      }
    }
    if (best < 1 && a.patch != b.patch) {
      for (const auto& cc : cross_corners[a.patch][b.patch]) {
        if (element_at_corner(cc.corner_a, a.ix, a.iy, n) &&
            element_at_corner(cc.corner_b, b.ix, b.iy, n)) {
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

  int resolved_far(int far_order) const { return far_order > 0 ? far_order : degree + 2; }
  int resolved_sing(int sing_order) const { return sing_order > 0 ? sing_order : degree + 3; }
};

// ------------------------------------------------------- pair integration
// operators.hpp:16-20; pair_integration.hpp:22-28
inline double laplace_g(double r) { return 1.0 / (4.0 * M_PI * r); }
inline cplx helmholtz_g(double r, cplx kappa) {
  return std::exp(cplx(0, -1) * kappa * r) / (4.0 * M_PI * r);
}
template <typename S>
inline S kernel_g(const Disc& d, double r) {
  if constexpr (std::is_same_v<S, double>)
    return laplace_g(r);
  else
    return helmholtz_g(r, d.kappa);
}

// dense column-major matrix
template <typename S>
struct Mat {
  int r = 0, c = 0;
  std::vector<S> a;
  Mat() = default;
  Mat(int rr, int cc) : r(rr), c(cc), a(static_cast<size_t>(rr) * cc, S(0)) {}
  S& operator()(int i, int j) { return a[i + static_cast<size_t>(r) * j]; }
  const S& operator()(int i, int j) const { return a[i + static_cast<size_t>(r) * j]; }
};

// pair_integration.hpp:32-73
template <typename S>
struct FarCache {
  std::vector<V3> pts;
  Mat<S> value;                 // nn x nl
  std::array<Mat<S>, 3> field;  // Maxwell
  Mat<S> dive;
};
template <typename S>
FarCache<S> make_far_cache(const Disc& d, int e, int n) {
  const auto& rule = gauss_rule(n);
  const auto& el = d.elements[e];
  const int nl = d.n_local, nn = n * n;
  FarCache<S> c;
  c.pts.resize(nn);
  if (d.is_vector()) {
    for (auto& f : c.field) f = Mat<S>(nn, nl);
    c.dive = Mat<S>(nn, nl);
  } else {
    c.value = Mat<S>(nn, nl);
  }
  Shapes s;
  int idx = 0;
  for (int b = 0; b < n; ++b)
    for (int a = 0; a < n; ++a, ++idx) {
      const double ul = rule.nodes[a], vl = rule.nodes[b];
      const Frame f = d.geom->frame(el.patch, el.ox + el.h * ul, el.oy + el.h * vl);
      const double w = rule.weights[a] * rule.weights[b] * f.sqrt_g * el.h * el.h;
      d.sample_shapes(e, ul, vl, s);
      c.pts[idx] = f.x;
      for (int l = 0; l < nl; ++l) {
        if (d.is_vector()) {
          for (int k = 0; k < 3; ++k) c.field[k](idx, l) = S(w * s.field[k][l]);
          c.dive(idx, l) = S(w * s.div[l]);
        } else {
          c.value(idx, l) = S(w * s.value[l]);
        }
      }
    }
  return c;
}

// A^T (K B) with K na x nb, A na x nl, B nb x nl
template <typename S>
static void atkb(const Mat<S>& A, const Mat<S>& K, const Mat<S>& B, S scale, Mat<S>& out) {
  const int na = K.r, nb = K.c, nl = A.c;
  Mat<S> kb(na, nl);
  for (int l = 0; l < nl; ++l)
    for (int j = 0; j < nb; ++j) {
      const S bj = B(j, l);
      for (int i = 0; i < na; ++i) kb(i, l) += K(i, j) * bj;
    }
  for (int lb = 0; lb < nl; ++lb)
    for (int la = 0; la < nl; ++la) {
      S acc(0);
      for (int i = 0; i < na; ++i) acc += A(i, la) * kb(i, lb);
      out(la, lb) += scale * acc;
    }
}

// pair_integration.hpp:76-95
template <typename S>
Mat<S> far_block(const Disc& d, const FarCache<S>& a, const FarCache<S>& b) {
  const int na = static_cast<int>(a.pts.size()), nb = static_cast<int>(b.pts.size());
  const int nl = d.n_local;
  Mat<S> k(na, nb);
  for (int j = 0; j < nb; ++j)
    for (int i = 0; i < na; ++i) k(i, j) = kernel_g<S>(d, norm(a.pts[i] - b.pts[j]));
  Mat<S> blk(nl, nl);
  if (!d.is_vector()) {
    atkb(a.value, k, b.value, S(1), blk);
    return blk;
  }
  if constexpr (!std::is_same_v<S, double>) {
    const cplx inv_k2 = 1.0 / (d.kappa * d.kappa);
    atkb(a.dive, k, b.dive, S(-inv_k2), blk);
    for (int c = 0; c < 3; ++c) atkb(a.field[c], k, b.field[c], S(1), blk);
  }
  return blk;
}

// pair_integration.hpp:98-134
template <typename S>
Mat<S> singular_block(const Disc& d, int ea, int eb, const PairInfo& info, int n) {
  const auto& rule = pair_rule(info.cls, n);
  const auto& ela = d.elements[ea];
  const auto& elb = d.elements[eb];
  const int nl = d.n_local;
  const bool vec = d.is_vector();
  const double h4 = ela.h * ela.h * elb.h * elb.h;
  const cplx inv_k2 = vec ? 1.0 / (d.kappa * d.kappa) : cplx(0);
  Mat<S> blk(nl, nl);
  Shapes sa, sb;
  for (const auto& p : rule) {
    double ua = p.ua, va = p.va, ub = p.ub, vb = p.vb;
    info.map_a.apply(ua, va);
    info.map_b.apply(ub, vb);
    const Frame fa = d.geom->frame(ela.patch, ela.ox + ela.h * ua, ela.oy + ela.h * va);
    const Frame fb = d.geom->frame(elb.patch, elb.ox + elb.h * ub, elb.oy + elb.h * vb);
    const double r = std::max(norm(fa.x - fb.x), 1e-14);
    const S g = kernel_g<S>(d, r);
    const double w = p.w * fa.sqrt_g * fb.sqrt_g * h4;
    d.sample_shapes(ea, ua, va, sa);
    d.sample_shapes(eb, ub, vb, sb);
    if constexpr (std::is_same_v<S, cplx>) {
      if (vec) {
        const cplx gw = g * w, gwk = g * w * inv_k2;
        for (int j = 0; j < nl; ++j)
          for (int i = 0; i < nl; ++i) {
            const double dots = sa.field[0][i] * sb.field[0][j] + sa.field[1][i] * sb.field[1][j] +
                                sa.field[2][i] * sb.field[2][j];
            const double divs = sa.div[i] * sb.div[j];
            blk(i, j) += gw * cplx(dots) - gwk * cplx(divs);
          }
        continue;
      }
    }
    const S gw = g * w;
    for (int j = 0; j < nl; ++j)
      for (int i = 0; i < nl; ++i) blk(i, j) += gw * S(sa.value[i] * sb.value[j]);
  }
  return blk;
}

// pair_integration.hpp:139-148
template <typename S>
Mat<S> pair_block(const Disc& d, const std::vector<FarCache<S>>& caches, int ea, int eb, int nsing) {
  const PairInfo info = d.classify_pair(ea, eb);
  if (info.cls == kFar) return far_block(d, caches[ea], caches[eb]);
  if (ea <= eb) return singular_block<S>(d, ea, eb, info, nsing);
  Mat<S> t = singular_block<S>(d, eb, ea, d.classify_pair(eb, ea), nsing);
  Mat<S> out(t.c, t.r);
  for (int j = 0; j < t.c; ++j)
    for (int i = 0; i < t.r; ++i) out(j, i) = t(i, j);
  return out;
}

// assembly.cpp:16-53 (dense Galerkin matrix, column-major nd x nd)
template <typename S>
void assemble_dense(const Disc& d, int far_order, int sing_order, S* A) {
  const int ne = d.ne(), nl = d.n_local, nd = d.n_dofs;
  const int nfar = d.resolved_far(far_order), nsing = d.resolved_sing(sing_order);
  std::vector<FarCache<S>> caches(ne);
#pragma omp parallel for schedule(static)
  for (int e = 0; e < ne; ++e) caches[e] = make_far_cache<S>(d, e, nfar);
  std::fill(A, A + static_cast<size_t>(nd) * nd, S(0));
  constexpr int kChunk = 32;
  std::vector<Mat<S>> buf(kChunk);
  for (int base = 0; base < ne; base += kChunk) {
    const int hi = std::min(base + kChunk, ne);
#pragma omp parallel for schedule(dynamic)
    for (int ea = base; ea < hi; ++ea) {
      Mat<S> rows(nl, nd);
      for (int eb = 0; eb < ne; ++eb) {
        const Mat<S> blk = pair_block<S>(d, caches, ea, eb, nsing);
        for (int lb = 0; lb < nl; ++lb) {
          const int col = d.l2g[static_cast<size_t>(eb) * nl + lb];
          const double sg = d.lsign[static_cast<size_t>(eb) * nl + lb];
          for (int la = 0; la < nl; ++la) rows(la, col) += sg * blk(la, lb);
        }
      }
      buf[ea - base] = std::move(rows);
    }
    for (int ea = base; ea < hi; ++ea)
      for (int la = 0; la < nl; ++la) {
        const int row = d.l2g[static_cast<size_t>(ea) * nl + la];
        const double sg = d.lsign[static_cast<size_t>(ea) * nl + la];
        for (int c = 0; c < nd; ++c) A[row + static_cast<size_t>(nd) * c] += sg * buf[ea - base](la, c);
      }
  }
}

// ---------------------------------------------------------------------- H2
// h2.cpp:13-45
static std::vector<double> cheb_nodes(int m) {
  std::vector<double> x(m);
  for (int k = 0; k < m; ++k) x[k] = 0.5 * (1.0 - std::cos(M_PI * k / (m - 1)));
  return x;
}
static std::vector<double> cheb_bary_weights(int m) {
  std::vector<double> w(m);
  for (int k = 0; k < m; ++k) {
    w[k] = (k % 2 == 0) ? 1.0 : -1.0;
    if (k == 0 || k == m - 1) w[k] *= 0.5;
  }
  return w;
}
static void lagrange_all(const std::vector<double>& nodes, const std::vector<double>& bw, double x,
                         double* out) {
  const int m = static_cast<int>(nodes.size());
  for (int k = 0; k < m; ++k) out[k] = 0.0;
  for (int k = 0; k < m; ++k)
    if (x == nodes[k]) {
      out[k] = 1.0;
      return;
    }
  double denom = 0;
  for (int k = 0; k < m; ++k) {
    out[k] = bw[k] / (x - nodes[k]);
    denom += out[k];
  }
  for (int k = 0; k < m; ++k) out[k] /= denom;
}

struct ClusterNode {  // h2.hpp:17-21
  int patch, level, sx, sy;
  Box box;
};
struct ClusterTree {  // h2.hpp:25-47, h2.cpp:49-90
  const Disc* disc = nullptr;
  int depth = 0, npp = 0;
  std::vector<int> level_offset;
  std::vector<ClusterNode> nodes;
  int node_id(int p, int l, int sx, int sy) const { return p * npp + level_offset[l] + sx + (1 << l) * sy; }
  int child(int id, int k) const {
    const auto& nd = nodes[id];
    if (nd.level >= depth) throw std::logic_error("ClusterTree::child: leaf node");
    return node_id(nd.patch, nd.level + 1, 2 * nd.sx + (k & 1), 2 * nd.sy + (k >> 1));
  }
  bool is_leaf(int id) const { return nodes[id].level == depth; }
  int leaf_element(int id) const {
    const auto& nd = nodes[id];
    if (nd.level != depth) throw std::logic_error("ClusterTree::leaf_element: not a leaf");
    return disc->element_index(nd.patch, nd.sx, nd.sy);
  }
  int root(int p) const { return p * npp; }
  explicit ClusterTree(const Disc& d) : disc(&d) {
    depth = d.level;
    level_offset.resize(depth + 1);
    npp = 0;
    for (int l = 0; l <= depth; ++l) {
      level_offset[l] = npp;
      npp += (1 << l) * (1 << l);
    }
    const int np = d.geom->patch_count();
    nodes.resize(static_cast<size_t>(np) * npp);
    for (int p = 0; p < np; ++p)
      for (int l = depth; l >= 0; --l) {
        const int n = 1 << l;
        for (int sy = 0; sy < n; ++sy)
          for (int sx = 0; sx < n; ++sx) {
            ClusterNode& nd = nodes[node_id(p, l, sx, sy)];
            nd.patch = p;
            nd.level = l;
            nd.sx = sx;
            nd.sy = sy;
            if (l == depth) {
              nd.box = d.elements[d.element_index(p, sx, sy)].box;
            } else {
              nd.box.set_empty();
              for (int k = 0; k < 4; ++k) nd.box.extend(nodes[child(node_id(p, l, sx, sy), k)].box);
            }
          }
      }
  }
};
bool admissible(const ClusterNode& a, const ClusterNode& b, double eta) {  // h2.cpp:92-97
  const double da = a.box.diag_norm();
  const double db = b.box.diag_norm();
  const double dist = a.box.exterior_distance(b.box);
  return std::max(da, db) <= eta * dist;
}

struct H2Base {
  virtual ~H2Base() = default;
};

template <typename S>
struct H2 : H2Base {
  const Disc* disc;
  int m;
  double eta;
  int far_order, sing_order;
  ClusterTree tree;
  int dim, nch;
  Mat<S> tl, tr;
  std::vector<Mat<S>> moments;  // per element, nch*m^2 x nl
  std::vector<std::pair<int, int>> near_pairs, far_pairs;
  std::vector<Mat<S>> near_blk;
  std::vector<Mat<S>> coupling;
  std::vector<int> near_row_start, far_row_start;
  std::vector<std::vector<V3>> images;

  // h2.cpp:99-129; flags bit0: skip near quadrature (zero blocks), bit1: skip couplings,
  // bit2: couplings evaluated where used (never stored; same formula, bitwise
  // equal), bit3: near blocks integrated where used (never stored) -- bits 2/3
  // let probe() check full-size configurations whose operator does not fit
  H2(const Disc& d, int m_, double eta_, int fo, int so, int flags)
      : disc(&d), m(m_), eta(eta_), far_order(fo), sing_order(so), tree(d), dim(d.n_dofs) {
    if (m < 2) throw std::invalid_argument("H2Matrix: interpolation degree m < 2");
    if (eta <= 0) throw std::invalid_argument("H2Matrix: eta must be positive");
    if constexpr (std::is_same_v<S, double>) {
      if (d.is_complex()) throw std::invalid_argument("H2Matrix<double>: complex kind");
    } else {
      if (!d.is_complex()) throw std::invalid_argument("H2Matrix<complex>: Laplace kind");
    }
    nch = d.is_vector() ? 4 : 1;
    const auto xi = cheb_nodes(m);
    const auto bw = cheb_bary_weights(m);
    tl = Mat<S>(m, m);
    tr = Mat<S>(m, m);
    std::vector<double> ll(m), lr(m);
    for (int j = 0; j < m; ++j) {
      lagrange_all(xi, bw, 0.5 * xi[j], ll.data());
      lagrange_all(xi, bw, 0.5 + 0.5 * xi[j], lr.data());
      for (int i = 0; i < m; ++i) {
        tl(i, j) = S(ll[i]);
        tr(i, j) = S(lr[i]);
      }
    }
    build_moments();
    build_blocks(flags);
  }

  void build_moments() {  // h2.cpp:131-173
    const int ne = disc->ne(), nl = disc->n_local;
    const auto xi = cheb_nodes(m);
    const auto bw = cheb_bary_weights(m);
    const int nq = disc->resolved_far(far_order);
    const auto& rule = gauss_rule(nq);
    const bool vec = disc->is_vector();
    moments.resize(ne);
#pragma omp parallel for schedule(static)
    for (int e = 0; e < ne; ++e) {
      const auto& el = disc->elements[e];
      Mat<double> mom(nch * m * m, nl);
      Shapes s;
      std::vector<double> lu(m), lv(m);
      for (int b = 0; b < nq; ++b)
        for (int a = 0; a < nq; ++a) {
          const double ul = rule.nodes[a], vl = rule.nodes[b];
          const Frame f = disc->geom->frame(el.patch, el.ox + el.h * ul, el.oy + el.h * vl);
          const double w = rule.weights[a] * rule.weights[b] * f.sqrt_g * el.h * el.h;
          disc->sample_shapes(e, ul, vl, s);
          lagrange_all(xi, bw, ul, lu.data());
          lagrange_all(xi, bw, vl, lv.data());
          for (int iv = 0; iv < m; ++iv)
            for (int iu = 0; iu < m; ++iu) {
              const double lw = w * lu[iu] * lv[iv];
              const int nu = iu + m * iv;
              for (int l = 0; l < nl; ++l) {
                if (vec) {
                  for (int dd = 0; dd < 3; ++dd) mom(dd * m * m + nu, l) += lw * s.field[dd][l];
                  mom(3 * m * m + nu, l) += lw * s.div[l];
                } else {
                  mom(nu, l) += lw * s.value[l];
                }
              }
            }
        }
      Mat<S> ms(mom.r, mom.c);
      for (size_t i = 0; i < mom.a.size(); ++i) ms.a[i] = S(mom.a[i]);
      moments[e] = std::move(ms);
    }
  }

  void build_blocks(int flags) {  // h2.cpp:175-252
    const int mm = m * m;
    const auto xi = cheb_nodes(m);
    const int np = disc->geom->patch_count();
    const int nn = static_cast<int>(tree.nodes.size());
    images.assign(nn, std::vector<V3>(mm));
#pragma omp parallel for schedule(static)
    for (int id = 0; id < nn; ++id) {
      const auto& nd = tree.nodes[id];
      const double hs = 1.0 / (1 << nd.level);
      for (int iv = 0; iv < m; ++iv)
        for (int iu = 0; iu < m; ++iu)
          images[id][iu + m * iv] =
              eval_patch(disc->geom->patches[nd.patch], hs * (nd.sx + xi[iu]), hs * (nd.sy + xi[iv])).x;
    }
    // dual traversal (h2.cpp:198-213)
    std::vector<std::pair<int, int>> stack;
    auto traverse = [&](auto&& self, int a, int b) -> void {
      if (admissible(tree.nodes[a], tree.nodes[b], eta)) {
        far_pairs.emplace_back(a, b);
        return;
      }
      if (tree.is_leaf(a)) {
        near_pairs.emplace_back(tree.leaf_element(a), tree.leaf_element(b));
        return;
      }
      for (int ka = 0; ka < 4; ++ka)
        for (int kb = 0; kb < 4; ++kb) self(self, tree.child(a, ka), tree.child(b, kb));
    };
    for (int pa = 0; pa < np; ++pa)
      for (int pb = 0; pb < np; ++pb) traverse(traverse, tree.root(pa), tree.root(pb));
    std::sort(near_pairs.begin(), near_pairs.end());
    std::sort(far_pairs.begin(), far_pairs.end());

    lazy_far = (flags & 4) != 0;
    lazy_near = (flags & 8) != 0;
    near_row_start.assign(disc->ne() + 1, 0);
    for (const auto& pr : near_pairs) ++near_row_start[pr.first + 1];
    for (int e = 0; e < disc->ne(); ++e) near_row_start[e + 1] += near_row_start[e];
    far_row_start.assign(nn + 1, 0);
    for (const auto& pr : far_pairs) ++far_row_start[pr.first + 1];
    for (int t = 0; t < nn; ++t) far_row_start[t + 1] += far_row_start[t];
    if (!lazy_far) coupling.resize(far_pairs.size());
#pragma omp parallel for schedule(dynamic, 64)
    for (size_t q = 0; q < coupling.size(); ++q) {
      Mat<S> k(mm, mm);
      if (!(flags & 2)) k = make_coupling(q);
      coupling[q] = std::move(k);
    }
    if (lazy_near) return;
    const int nfar = disc->resolved_far(far_order);
    const int nsing = disc->resolved_sing(sing_order);
    const int ne = disc->ne();
    std::vector<FarCache<S>> caches(ne);
    if (!(flags & 1)) {
#pragma omp parallel for schedule(static)
      for (int e = 0; e < ne; ++e) caches[e] = make_far_cache<S>(*disc, e, nfar);
    }
    near_blk.resize(near_pairs.size());
#pragma omp parallel for schedule(dynamic, 16)
    for (size_t q = 0; q < near_pairs.size(); ++q) {
      const auto [ea, eb] = near_pairs[q];
      if (flags & 1)
        near_blk[q] = Mat<S>(disc->n_local, disc->n_local);
      else
        near_blk[q] = pair_block<S>(*disc, caches, ea, eb, nsing);
    }
  }

  bool lazy_far = false, lazy_near = false;
  // K[nu, mu] = G(|img_ta[nu] - img_tb[mu]|) (h2.cpp:218-229)
  Mat<S> make_coupling(size_t q) const {
    const int mm = m * m;
    const auto [ta, tb] = far_pairs[q];
    Mat<S> k(mm, mm);
    for (int mu = 0; mu < mm; ++mu)
      for (int nu = 0; nu < mm; ++nu) k(nu, mu) = kernel_g<S>(*disc, norm(images[ta][nu] - images[tb][mu]));
    return k;
  }
  const Mat<S>& coupling_at(size_t q, Mat<S>& tmp) const {
    if (!lazy_far) return coupling[q];
    tmp = make_coupling(q);
    return tmp;
  }
  // near block of pair q (stored, or integrated now: h2.cpp:236-243)
  Mat<S> near_block_at(size_t q) const {
    if (!lazy_near) return near_blk[q];
    const auto [ea, eb] = near_pairs[q];
    thread_local std::vector<FarCache<S>> caches;  // per thread, only the pair's two entries filled
    if (caches.size() != static_cast<size_t>(disc->ne())) caches.assign(disc->ne(), FarCache<S>{});
    const int nfar = disc->resolved_far(far_order);
    caches[ea] = make_far_cache<S>(*disc, ea, nfar);
    if (eb != ea) caches[eb] = make_far_cache<S>(*disc, eb, nfar);
    Mat<S> b = pair_block<S>(*disc, caches, ea, eb, disc->resolved_sing(sing_order));
    caches[ea] = FarCache<S>{};
    caches[eb] = FarCache<S>{};
    return b;
  }

  // h2.cpp:254-378; optional outputs: up (phase 3), down after the far field
  // (phase 4) and after the downward pass (phase 5), each [node][c*m^2 + nu]
  void apply(const S* x, S* y, S* up_out = nullptr, S* down4_out = nullptr, S* down5_out = nullptr) const {
    const int mm = m * m;
    const int ne = disc->ne(), nl = disc->n_local;
    const int nn = static_cast<int>(tree.nodes.size());
    const int depth = tree.depth;
    const int np = disc->geom->patch_count();
    const bool vec = disc->is_vector();
    S divw(0);
    if constexpr (std::is_same_v<S, cplx>) {
      if (vec) divw = -1.0 / (disc->kappa * disc->kappa);
    }
    std::vector<S> coef(static_cast<size_t>(ne) * nl);
#pragma omp parallel for schedule(static)
    for (int e = 0; e < ne; ++e)
      for (int l = 0; l < nl; ++l) {
        const size_t i = static_cast<size_t>(e) * nl + l;
        coef[i] = S(disc->lsign[i]) * x[disc->l2g[i]];
      }
    const int ncol = mm * nch;
    std::vector<S> up(static_cast<size_t>(nn) * ncol, S(0));
#pragma omp parallel for schedule(static)
    for (int id = 0; id < nn; ++id) {
      if (!tree.is_leaf(id)) continue;
      const int e = tree.leaf_element(id);
      const Mat<S>& mo = moments[e];
      for (int r = 0; r < mo.r; ++r) {
        S acc(0);
        for (int l = 0; l < nl; ++l) acc += mo(r, l) * coef[static_cast<size_t>(e) * nl + l];
        up[static_cast<size_t>(id) * ncol + r] = acc;
      }
    }
    // Y += tu X tv^T on m x m column-major views
    auto add_tx = [&](const Mat<S>& tu, const Mat<S>& tv, const S* X, S* Y, bool transpose) {
      // transpose=false: Y += tu * X * tv^T ; true: Y += tu^T * X * tv
      std::vector<S> tmp(mm, S(0));
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) {
          const S xk = X[k + m * j];
          for (int i = 0; i < m; ++i) tmp[i + m * j] += (transpose ? tu(k, i) : tu(i, k)) * xk;
        }
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) {
          const S t = transpose ? tv(k, j) : tv(j, k);
          for (int i = 0; i < m; ++i) Y[i + m * j] += tmp[i + m * k] * t;
        }
    };
    for (int l = depth - 1; l >= 0; --l) {
      const int n = 1 << l;
#pragma omp parallel for schedule(static) collapse(2)
      for (int p = 0; p < np; ++p)
        for (int s = 0; s < n * n; ++s) {
          const int id = tree.node_id(p, l, s % n, s / n);
          S* Y = &up[static_cast<size_t>(id) * ncol];
          for (int k = 0; k < 4; ++k) {
            const S* X = &up[static_cast<size_t>(tree.child(id, k)) * ncol];
            const Mat<S>& tu = (k & 1) ? tr : tl;
            const Mat<S>& tv = (k >> 1) ? tr : tl;
            for (int c = 0; c < nch; ++c) add_tx(tu, tv, X + c * mm, Y + c * mm, false);
          }
        }
    }
    std::vector<S> down(static_cast<size_t>(nn) * ncol, S(0));
    std::vector<char> has_down(nn, 0);
#pragma omp parallel for schedule(dynamic)
    for (int t = 0; t < nn; ++t) {
      if (far_row_start[t] == far_row_start[t + 1]) continue;
      has_down[t] = 1;
      S* acc = &down[static_cast<size_t>(t) * ncol];
      Mat<S> ktmp;
      for (int q = far_row_start[t]; q < far_row_start[t + 1]; ++q) {
        const Mat<S>& K = coupling_at(q, ktmp);
        const S* src = &up[static_cast<size_t>(far_pairs[q].second) * ncol];
        for (int c = 0; c < nch; ++c) {
          const S w = (vec && c == 3) ? divw : S(1);
          std::vector<S> kx(mm, S(0));
          for (int mu = 0; mu < mm; ++mu) {
            const S xm = src[c * mm + mu];
            for (int nu = 0; nu < mm; ++nu) kx[nu] += K(nu, mu) * xm;
          }
          for (int nu = 0; nu < mm; ++nu) acc[c * mm + nu] += w * kx[nu];
        }
      }
    }
    if (up_out) std::copy(up.begin(), up.end(), up_out);
    if (down4_out) std::copy(down.begin(), down.end(), down4_out);
    for (int l = 0; l < depth; ++l) {
      const int n = 2 << l;
#pragma omp parallel for schedule(static) collapse(2)
      for (int p = 0; p < np; ++p)
        for (int s = 0; s < n * n; ++s) {
          const int sx = s % n, sy = s / n;
          const int parent = tree.node_id(p, l, sx / 2, sy / 2);
          if (!has_down[parent]) continue;
          const int id = tree.node_id(p, l + 1, sx, sy);
          has_down[id] = 1;
          const Mat<S>& tu = (sx & 1) ? tr : tl;
          const Mat<S>& tv = (sy & 1) ? tr : tl;
          for (int c = 0; c < nch; ++c)
            add_tx(tu, tv, &down[static_cast<size_t>(parent) * ncol + c * mm],
                   &down[static_cast<size_t>(id) * ncol + c * mm], true);
        }
    }
    if (down5_out) std::copy(down.begin(), down.end(), down5_out);
    std::vector<S> near_rows(static_cast<size_t>(ne) * nl, S(0));
#pragma omp parallel for schedule(dynamic)
    for (int e = 0; e < ne; ++e) {
      S* acc = &near_rows[static_cast<size_t>(e) * nl];
      for (int q = near_row_start[e]; q < near_row_start[e + 1]; ++q) {
        const Mat<S> B = near_block_at(q);
        const S* c = &coef[static_cast<size_t>(near_pairs[q].second) * nl];
        for (int lb = 0; lb < nl; ++lb)
          for (int la = 0; la < nl; ++la) acc[la] += B(la, lb) * c[lb];
      }
    }
    std::fill(y, y + dim, S(0));
    for (int p = 0; p < np; ++p) {
      const int n = 1 << depth;
      for (int sy = 0; sy < n; ++sy)
        for (int sx = 0; sx < n; ++sx) {
          const int id = tree.node_id(p, depth, sx, sy);
          const int e = tree.leaf_element(id);
          std::vector<S> loc(near_rows.begin() + static_cast<size_t>(e) * nl,
                             near_rows.begin() + static_cast<size_t>(e + 1) * nl);
          if (has_down[id]) {
            const Mat<S>& mo = moments[e];
            const S* dn = &down[static_cast<size_t>(id) * ncol];
            for (int l = 0; l < nl; ++l) {
              S acc(0);
              for (int r = 0; r < mo.r; ++r) acc += mo(r, l) * dn[r];
              loc[l] += acc;
            }
          }
          for (int l = 0; l < nl; ++l) {
            const size_t i = static_cast<size_t>(e) * nl + l;
            y[disc->l2g[i]] += S(disc->lsign[i]) * loc[l];
          }
        }
    }
  }

  // Selected outputs of apply() without the full operator: up (all nodes), the
  // phase-4 down of `nodes`, and y at `dofs`.  Only what they depend on is
  // evaluated -- the full upward pass, the far rows of the selected nodes and of
  // the ancestors of the selected DOFs' leaves, the near rows of their elements
  // -- with apply()'s arithmetic in apply()'s order, so every value equals
  // apply()'s bitwise.  With lazy couplings / near blocks (flags bits 2, 3) this
  // checks full-size configurations whose operator does not fit host memory.
  void probe(const S* x, S* up_out, int n_nodes, const int* nodes, S* down4_out, int n_dofs, const int* dofs,
             S* y_out) const {
    const int mm = m * m, ncol = mm * nch;
    const int ne = disc->ne(), nl = disc->n_local, nn = static_cast<int>(tree.nodes.size());
    const int depth = tree.depth, np = disc->geom->patch_count();
    const bool vec = disc->is_vector();
    S divw(0);
    if constexpr (std::is_same_v<S, cplx>) {
      if (vec) divw = -1.0 / (disc->kappa * disc->kappa);
    }
    std::vector<S> coef(static_cast<size_t>(ne) * nl);
#pragma omp parallel for schedule(static)
    for (int e = 0; e < ne; ++e)
      for (int l = 0; l < nl; ++l) {
        const size_t i = static_cast<size_t>(e) * nl + l;
        coef[i] = S(disc->lsign[i]) * x[disc->l2g[i]];
      }
    std::vector<S> up(static_cast<size_t>(nn) * ncol, S(0));
#pragma omp parallel for schedule(static)
    for (int id = 0; id < nn; ++id) {
      if (!tree.is_leaf(id)) continue;
      const int e = tree.leaf_element(id);
      const Mat<S>& mo = moments[e];
      for (int r = 0; r < mo.r; ++r) {
        S acc(0);
        for (int l = 0; l < nl; ++l) acc += mo(r, l) * coef[static_cast<size_t>(e) * nl + l];
        up[static_cast<size_t>(id) * ncol + r] = acc;
      }
    }
    auto add_tx = [&](const Mat<S>& tu, const Mat<S>& tv, const S* X, S* Y, bool transpose) {
      std::vector<S> tmp(mm, S(0));
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) {
          const S xk = X[k + m * j];
          for (int i = 0; i < m; ++i) tmp[i + m * j] += (transpose ? tu(k, i) : tu(i, k)) * xk;
        }
      for (int j = 0; j < m; ++j)
        for (int k = 0; k < m; ++k) {
          const S t = transpose ? tv(k, j) : tv(j, k);
          for (int i = 0; i < m; ++i) Y[i + m * j] += tmp[i + m * k] * t;
        }
    };
    for (int l = depth - 1; l >= 0; --l) {
      const int n = 1 << l;
#pragma omp parallel for schedule(static) collapse(2)
      for (int p = 0; p < np; ++p)
        for (int sq = 0; sq < n * n; ++sq) {
          const int id = tree.node_id(p, l, sq % n, sq / n);
          S* Y = &up[static_cast<size_t>(id) * ncol];
          for (int k = 0; k < 4; ++k) {
            const S* X = &up[static_cast<size_t>(tree.child(id, k)) * ncol];
            const Mat<S>& tu = (k & 1) ? tr : tl;
            const Mat<S>& tv = (k >> 1) ? tr : tl;
            for (int c = 0; c < nch; ++c) add_tx(tu, tv, X + c * mm, Y + c * mm, false);
          }
        }
    }
    if (up_out) std::copy(up.begin(), up.end(), up_out);
    // phase-4 row of node t (the far loop of apply())
    auto down4 = [&](int t, S* acc) {
      for (int i = 0; i < ncol; ++i) acc[i] = S(0);
      Mat<S> ktmp;
      for (int q = far_row_start[t]; q < far_row_start[t + 1]; ++q) {
        const Mat<S>& K = coupling_at(q, ktmp);
        const S* src = &up[static_cast<size_t>(far_pairs[q].second) * ncol];
        for (int c = 0; c < nch; ++c) {
          const S w = (vec && c == 3) ? divw : S(1);
          std::vector<S> kx(mm, S(0));
          for (int mu = 0; mu < mm; ++mu) {
            const S xm = src[c * mm + mu];
            for (int nu = 0; nu < mm; ++nu) kx[nu] += K(nu, mu) * xm;
          }
          for (int nu = 0; nu < mm; ++nu) acc[c * mm + nu] += w * kx[nu];
        }
      }
    };
#pragma omp parallel for schedule(dynamic)
    for (int k = 0; k < n_nodes; ++k) down4(nodes[k], down4_out + static_cast<size_t>(k) * ncol);
    if (n_dofs == 0) return;
    // elements touching the selected DOFs, ascending (apply()'s gather order)
    std::vector<int> pos(disc->n_dofs, -1);
    for (int k = 0; k < n_dofs; ++k) pos[dofs[k]] = k;
    std::vector<int> els;
    for (int e = 0; e < ne; ++e)
      for (int l = 0; l < nl; ++l)
        if (pos[disc->l2g[static_cast<size_t>(e) * nl + l]] >= 0) {
          els.push_back(e);
          break;
        }
    const int side = 1 << depth;
    std::vector<std::vector<S>> loc(els.size());
#pragma omp parallel for schedule(dynamic)
    for (size_t i = 0; i < els.size(); ++i) {
      const int e = els[i];
      const int p = e / (side * side), sxe = e % side, sye = (e / side) % side;
      // down along the root -> leaf path (apply()'s phase 5 restricted to it)
      std::vector<S> dpar(ncol), dch(ncol);
      int parent = tree.node_id(p, 0, 0, 0);
      down4(parent, dpar.data());
      bool has = far_row_start[parent] < far_row_start[parent + 1];
      for (int l = 0; l < depth; ++l) {
        const int sh = depth - l - 1, sx = sxe >> sh, sy = sye >> sh;
        const int id = tree.node_id(p, l + 1, sx, sy);
        down4(id, dch.data());
        const bool own = far_row_start[id] < far_row_start[id + 1];
        if (has) {
          const Mat<S>& tu = (sx & 1) ? tr : tl;
          const Mat<S>& tv = (sy & 1) ? tr : tl;
          for (int c = 0; c < nch; ++c) add_tx(tu, tv, &dpar[c * mm], &dch[c * mm], true);
        }
        has = has || own;
        std::swap(dpar, dch);
      }
      std::vector<S> lc(nl, S(0));
      for (int q = near_row_start[e]; q < near_row_start[e + 1]; ++q) {
        const Mat<S> B = near_block_at(q);
        const S* c = &coef[static_cast<size_t>(near_pairs[q].second) * nl];
        for (int lb = 0; lb < nl; ++lb)
          for (int la = 0; la < nl; ++la) lc[la] += B(la, lb) * c[lb];
      }
      if (has) {
        const Mat<S>& mo = moments[e];
        for (int l = 0; l < nl; ++l) {
          S acc(0);
          for (int r = 0; r < mo.r; ++r) acc += mo(r, l) * dpar[r];
          lc[l] += acc;
        }
      }
      loc[i] = std::move(lc);
    }
    for (int k = 0; k < n_dofs; ++k) y_out[k] = S(0);
    for (size_t i = 0; i < els.size(); ++i)
      for (int l = 0; l < nl; ++l) {
        const size_t g = static_cast<size_t>(els[i]) * nl + l;
        const int k = pos[disc->l2g[g]];
        if (k >= 0) y_out[k] += S(disc->lsign[g]) * loc[i][l];
      }
  }

  void storage(long long* out) const {  // h2.cpp:380-390
    size_t ne_ = 0, fe = 0, mo = 0;
    for (const auto& b : near_blk) ne_ += b.a.size();
    for (const auto& k : coupling) fe += k.a.size();
    for (const auto& x : moments) mo += x.a.size();
    out[0] = static_cast<long long>(ne_);
    out[1] = static_cast<long long>(fe);
    out[2] = static_cast<long long>((ne_ + fe + mo + 2 * tl.a.size()) * sizeof(S));
  }
};

}  // namespace orc

// ============================================================== C interface
using namespace orc;

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
struct OH2 {
  Disc* disc;
  std::unique_ptr<H2<double>> real;
  std::unique_ptr<H2<cplx>> cx;
};
template <typename F>
void with_h2(void* hp, F&& f) {
  OH2* h = static_cast<OH2*>(hp);
  if (h->real) f(*h->real); else f(*h->cx);
}
}  // namespace

extern "C" {

int orc_last_error(char* buf, int n) {
  std::snprintf(buf, n, "%s", g_err.c_str());
  return static_cast<int>(g_err.size());
}

int orc_gauss(int n, double* nodes, double* weights) {
  return guard([&] {
    const auto& r = gauss_rule(n);
    for (int i = 0; i < n; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
  });
}

// writes 5 doubles per point (ua, va, ub, vb, w); returns count in *count
int orc_pair_rule(int cls, int n, double* out, long long* count) {
  return guard([&] {
    const auto& r = pair_rule(cls, n);
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

// geom: 0 = make_sphere(radius, center), 1 = make_square()
int orc_disc_create(int geom, double radius, const double* center, int kind, double kre, double kim,
                    int P, int rep, int L, void** out) {
  return guard([&] {
    auto g = std::make_shared<Geometry>(geom == 0 ? make_sphere(radius, V3(center[0], center[1], center[2]))
                                                  : make_square());
    *out = new Disc(std::move(g), kind, cplx(kre, kim), P, rep, L);
  });
}
void orc_disc_destroy(void* d) { delete static_cast<Disc*>(d); }

// out: dofs, ne, nl, np, level, degree, n_edges, n_vertices
void orc_disc_info(void* dp, int* out) {
  const Disc& d = *static_cast<Disc*>(dp);
  out[0] = d.n_dofs;
  out[1] = d.ne();
  out[2] = d.n_local;
  out[3] = d.geom->patch_count();
  out[4] = d.level;
  out[5] = d.degree;
  out[6] = static_cast<int>(d.geom->edges.size());
  out[7] = static_cast<int>(d.geom->vertices.size());
}
void orc_disc_l2g(void* dp, int* l2g, double* sign) {
  const Disc& d = *static_cast<Disc*>(dp);
  std::copy(d.l2g.begin(), d.l2g.end(), l2g);
  std::copy(d.lsign.begin(), d.lsign.end(), sign);
}
// ints: patch, ix, iy per element; dbl: h, ox, oy, min3, max3 per element
void orc_disc_elements(void* dp, int* ints, double* dbl) {
  const Disc& d = *static_cast<Disc*>(dp);
  for (int e = 0; e < d.ne(); ++e) {
    const auto& el = d.elements[e];
    ints[3 * e] = el.patch;
    ints[3 * e + 1] = el.ix;
    ints[3 * e + 2] = el.iy;
    double* o = dbl + 9 * e;
    o[0] = el.h;
    o[1] = el.ox;
    o[2] = el.oy;
    for (int k = 0; k < 3; ++k) {
      o[3 + k] = el.box.mn[k];
      o[6 + k] = el.box.mx[k];
    }
  }
}
// control data of patch p: degrees, knot vectors, homogeneous points
// sizes out: [pu, pv, nku, nkv]; if arrays non-null they are filled
void orc_patch(void* dp, int p, int* sizes, double* ku, double* kv, double* cw, double* w) {
  const Disc& d = *static_cast<Disc*>(dp);
  const Patch& s = d.geom->patches[p];
  sizes[0] = s.kv_u.degree;
  sizes[1] = s.kv_v.degree;
  sizes[2] = static_cast<int>(s.kv_u.knots.size());
  sizes[3] = static_cast<int>(s.kv_v.knots.size());
  if (ku) std::copy(s.kv_u.knots.begin(), s.kv_u.knots.end(), ku);
  if (kv) std::copy(s.kv_v.knots.begin(), s.kv_v.knots.end(), kv);
  if (cw) std::copy(s.cw.begin(), s.cw.end(), cw);
  if (w) std::copy(s.w.begin(), s.w.end(), w);
}
// edges: 5 ints each (patch_a, edge_a, patch_b, edge_b, reversed)
void orc_edges(void* dp, int* out) {
  const Disc& d = *static_cast<Disc*>(dp);
  int i = 0;
  for (const auto& e : d.geom->edges) {
    out[i++] = e.patch_a;
    out[i++] = e.edge_a;
    out[i++] = e.patch_b;
    out[i++] = e.edge_b;
    out[i++] = e.reversed ? 1 : 0;
  }
}
// frame: x3 du3 dv3 normal3 sqrt_g
int orc_frame(void* dp, int p, double u, double v, double* out) {
  return guard([&] {
    const Disc& d = *static_cast<Disc*>(dp);
    const Frame f = d.geom->frame(p, u, v);
    for (int k = 0; k < 3; ++k) {
      out[k] = f.x[k];
      out[3 + k] = f.du[k];
      out[6 + k] = f.dv[k];
      out[9 + k] = f.normal[k];
    }
    out[12] = f.sqrt_g;
  });
}
// value[nl] (scalar) or field[3*nl] row-major by component + div[nl]
int orc_sample_shapes(void* dp, int e, double u, double v, double* value, double* field, double* div) {
  return guard([&] {
    const Disc& d = *static_cast<Disc*>(dp);
    Shapes s;
    d.sample_shapes(e, u, v, s);
    for (int l = 0; l < d.n_local; ++l) {
      if (value) value[l] = s.value[l];
      if (field)
        for (int k = 0; k < 3; ++k) field[k * d.n_local + l] = s.field[k][l];
      if (div) div[l] = s.div[l];
    }
  });
}
// returns cls; maps: 6 ints (swap, flip_u, flip_v for a, then b)
int orc_classify(void* dp, int ea, int eb, int* maps) {
  const Disc& d = *static_cast<Disc*>(dp);
  const PairInfo info = d.classify_pair(ea, eb);
  if (maps) {
    maps[0] = info.map_a.swap; maps[1] = info.map_a.flip_u; maps[2] = info.map_a.flip_v;
    maps[3] = info.map_b.swap; maps[4] = info.map_b.flip_u; maps[5] = info.map_b.flip_v;
  }
  return info.cls;
}
// blocks for a list of element pairs, nl*nl column-major each, complex interleaved
int orc_pair_blocks(void* dp, const int* pairs, long long npairs, int far_order, int sing_order, double* out) {
  return guard([&] {
    const Disc& d = *static_cast<Disc*>(dp);
    const int nl = d.n_local, nfar = d.resolved_far(far_order), nsing = d.resolved_sing(sing_order);
    auto run = [&](auto tag) {
      using S = decltype(tag);
      std::vector<FarCache<S>> caches(d.ne());
      std::vector<char> need(d.ne(), 0);
      for (long long q = 0; q < npairs; ++q) need[pairs[2 * q]] = need[pairs[2 * q + 1]] = 1;
#pragma omp parallel for schedule(dynamic, 16)
      for (int e = 0; e < d.ne(); ++e)
        if (need[e]) caches[e] = make_far_cache<S>(d, e, nfar);
#pragma omp parallel for schedule(dynamic, 4)
      for (long long q = 0; q < npairs; ++q) {
        const Mat<S> b = pair_block<S>(d, caches, pairs[2 * q], pairs[2 * q + 1], nsing);
        std::memcpy(out + static_cast<size_t>(q) * nl * nl * (sizeof(S) / 8), b.a.data(), sizeof(S) * nl * nl);
      }
    };
    if (d.is_complex()) run(cplx{}); else run(double{});
  });
}
int orc_dense(void* dp, int far_order, int sing_order, double* A) {
  return guard([&] {
    const Disc& d = *static_cast<Disc*>(dp);
    if (d.is_complex())
      assemble_dense<cplx>(d, far_order, sing_order, reinterpret_cast<cplx*>(A));
    else
      assemble_dense<double>(d, far_order, sing_order, A);
  });
}

int orc_h2_create(void* dp, int m, double eta, int far_order, int sing_order, int flags, void** out) {
  return guard([&] {
    Disc* d = static_cast<Disc*>(dp);
    auto h = std::make_unique<OH2>();
    h->disc = d;
    if (d->is_complex())
      h->cx = std::make_unique<H2<cplx>>(*d, m, eta, far_order, sing_order, flags);
    else
      h->real = std::make_unique<H2<double>>(*d, m, eta, far_order, sing_order, flags);
    *out = h.release();
  });
}
void orc_h2_destroy(void* h) { delete static_cast<OH2*>(h); }

// out: near_count, far_count, node_count, near_entries, far_entries, total_bytes, nch, m
void orc_h2_info(void* hp, long long* out) {
  with_h2(hp, [&](auto& h) {
    out[0] = static_cast<long long>(h.near_pairs.size());
    out[1] = static_cast<long long>(h.far_pairs.size());
    out[2] = static_cast<long long>(h.tree.nodes.size());
    h.storage(out + 3);
    out[6] = h.nch;
    out[7] = h.m;
  });
}
void orc_h2_near_pairs(void* hp, int* out) {
  with_h2(hp, [&](auto& h) {
    for (size_t i = 0; i < h.near_pairs.size(); ++i) {
      out[2 * i] = h.near_pairs[i].first;
      out[2 * i + 1] = h.near_pairs[i].second;
    }
  });
}
void orc_h2_far_pairs(void* hp, int* out) {
  with_h2(hp, [&](auto& h) {
    for (size_t i = 0; i < h.far_pairs.size(); ++i) {
      out[2 * i] = h.far_pairs[i].first;
      out[2 * i + 1] = h.far_pairs[i].second;
    }
  });
}
void orc_h2_near_blocks(void* hp, long long first, long long count, double* out) {
  with_h2(hp, [&](auto& h) {
    using S = typename std::decay_t<decltype(h.tl.a)>::value_type;
    const int nl = h.disc->n_local;
    for (long long q = 0; q < count; ++q)
      std::memcpy(out + static_cast<size_t>(q) * nl * nl * (sizeof(S) / 8), h.near_blk[first + q].a.data(),
                  sizeof(S) * nl * nl);
  });
}
void orc_h2_couplings(void* hp, long long first, long long count, double* out) {
  with_h2(hp, [&](auto& h) {
    using S = typename std::decay_t<decltype(h.tl.a)>::value_type;
    const size_t n = static_cast<size_t>(h.m) * h.m * h.m * h.m;
    for (long long q = 0; q < count; ++q)
      std::memcpy(out + q * n * (sizeof(S) / 8), h.coupling[first + q].a.data(), sizeof(S) * n);
  });
}
void orc_h2_moments(void* hp, double* out) {
  with_h2(hp, [&](auto& h) {
    using S = typename std::decay_t<decltype(h.tl.a)>::value_type;
    size_t off = 0;
    for (const auto& mo : h.moments) {
      std::memcpy(out + off, mo.a.data(), sizeof(S) * mo.a.size());
      off += mo.a.size() * (sizeof(S) / 8);
    }
  });
}
void orc_h2_images(void* hp, double* out) {
  with_h2(hp, [&](auto& h) {
    size_t i = 0;
    for (const auto& img : h.images)
      for (const auto& p : img)
        for (int k = 0; k < 3; ++k) out[i++] = p[k];
  });
}
// node boxes: min3 max3 per node
void orc_h2_boxes(void* hp, double* out) {
  with_h2(hp, [&](auto& h) {
    for (size_t i = 0; i < h.tree.nodes.size(); ++i)
      for (int k = 0; k < 3; ++k) {
        out[6 * i + k] = h.tree.nodes[i].box.mn[k];
        out[6 * i + 3 + k] = h.tree.nodes[i].box.mx[k];
      }
  });
}
void orc_h2_transfer(void* hp, double* tl, double* tr) {
  with_h2(hp, [&](auto& h) {
    using S = typename std::decay_t<decltype(h.tl.a)>::value_type;
    std::memcpy(tl, h.tl.a.data(), sizeof(S) * h.tl.a.size());
    std::memcpy(tr, h.tr.a.data(), sizeof(S) * h.tr.a.size());
  });
}
int orc_h2_apply(void* hp, const double* x, double* y) {
  return guard([&] {
    OH2* h = static_cast<OH2*>(hp);
    if (h->real)
      h->real->apply(x, y);
    else
      h->cx->apply(reinterpret_cast<const cplx*>(x), reinterpret_cast<cplx*>(y));
  });
}
// apply with internals: up, down after phase 4, down after phase 5 (any may be null)
int orc_h2_apply_ex(void* hp, const double* x, double* y, double* up, double* down4, double* down5) {
  return guard([&] {
    OH2* h = static_cast<OH2*>(hp);
    if (h->real) {
      h->real->apply(x, y, up, down4, down5);
    } else {
      auto c = [](double* p) { return reinterpret_cast<cplx*>(p); };
      h->cx->apply(reinterpret_cast<const cplx*>(x), c(y), c(up), c(down4), c(down5));
    }
  });
}
// probe: up (all nodes), phase-4 down of `nodes`, y at `dofs` (see H2::probe)
int orc_h2_probe(void* hp, const double* x, double* up, int n_nodes, const int* nodes, double* down4, int n_dofs,
                 const int* dofs, double* y) {
  return guard([&] {
    OH2* h = static_cast<OH2*>(hp);
    if (h->real) {
      h->real->probe(x, up, n_nodes, nodes, down4, n_dofs, dofs, y);
    } else {
      auto c = [](double* p) { return reinterpret_cast<cplx*>(p); };
      h->cx->probe(reinterpret_cast<const cplx*>(x), c(up), n_nodes, nodes, c(down4), n_dofs, dofs, c(y));
    }
  });
}
int orc_admissible(const double* boxa, const double* boxb, double eta) {
  ClusterNode a{}, b{};
  for (int k = 0; k < 3; ++k) {
    a.box.mn[k] = boxa[k]; a.box.mx[k] = boxa[3 + k];
    b.box.mn[k] = boxb[k]; b.box.mx[k] = boxb[3 + k];
  }
  return admissible(a, b, eta) ? 1 : 0;
}

}  // extern "C"
