// Block partition on the device (setup on the GPU).
//
// The dual traversal of h2.cpp:198-216 runs level by level: every frontier
// pair (same-level nodes a, b) is decided far (admissible, h2.cpp:92-97), near
// (inadmissible leaves) or refined into its 16 child pairs; CUB scans compact
// the three outputs.  The admissibility test reproduces the host's (and the
// reference's) operation order exactly -- diagonals from the host, exterior
// distance with explicit round-to-nearest multiplies/adds and a correctly
// rounded square root, no contraction -- so the partition is bit-identical.
// The pair lists are then radix-sorted by (a, b) (the lexicographic order of
// h2.cpp:215-216), and the CSR row starts, upper starts and transposes of the
// symmetric admissible relation come from binary searches.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "igb_host.hpp"

namespace igb {
namespace {

#define IGB_PCUDA(call)                                                                                    \
  do {                                                                                                     \
    const cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)

struct DevBox {
  double mn[3], mx[3];
};

// decision of one same-level pair: 0 far, 1 near (leaf level), 2 refine
__global__ void k_decide(long long n, const int* __restrict__ pa, const int* __restrict__ pb,
                         const DevBox* __restrict__ box, const double* __restrict__ diag, double eta, int leaf,
                         unsigned char* __restrict__ dec, int* __restrict__ is_far, int* __restrict__ is_near,
                         int* __restrict__ is_ref) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int a = pa[i], b = pb[i];
  const DevBox A = box[a], B = box[b];
  double d2 = 0.0;  // Box::exterior_distance, term by term like the host
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (A.mn[k] > B.mx[k]) {
      const double aux = __dsub_rn(A.mn[k], B.mx[k]);
      d2 = __dadd_rn(d2, __dmul_rn(aux, aux));
    } else if (B.mn[k] > A.mx[k]) {
      const double aux = __dsub_rn(B.mn[k], A.mx[k]);
      d2 = __dadd_rn(d2, __dmul_rn(aux, aux));
    }
  }
  const double dist = __dsqrt_rn(d2);
  const unsigned char c = fmax(diag[a], diag[b]) <= __dmul_rn(eta, dist) ? 0 : (leaf ? 1 : 2);
  dec[i] = c;
  is_far[i] = c == 0;
  is_near[i] = c == 1;
  is_ref[i] = c == 2;
}

struct Level {
  int npp, off, off_next, side;  // nodes per patch, first node of this / next level, 2^level
};

__global__ void k_emit(long long n, const int* __restrict__ pa, const int* __restrict__ pb,
                       const unsigned char* __restrict__ dec, const int* __restrict__ far_pos,
                       const int* __restrict__ near_pos, const int* __restrict__ ref_pos, Level lv, int epp,
                       int n1, unsigned long long* __restrict__ far_keys, long long far_base,
                       unsigned long long* __restrict__ near_keys, int* __restrict__ na, int* __restrict__ nb) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int a = pa[i], b = pb[i];
  const unsigned char c = dec[i];
  if (c == 0) {
    far_keys[far_base + far_pos[i]] = (static_cast<unsigned long long>(a) << 32) | static_cast<unsigned>(b);
  } else if (c == 1) {  // leaves -> element ids (p * epp + sx + 2^L sy)
    auto el = [&](int node) {
      const int p = node / lv.npp, r = node % lv.npp - lv.off;
      return p * epp + (r % n1) + n1 * (r / n1);
    };
    near_keys[near_pos[i]] = (static_cast<unsigned long long>(el(a)) << 32) | static_cast<unsigned>(el(b));
  } else {
    auto child = [&](int node, int k) {
      const int p = node / lv.npp, r = node % lv.npp - lv.off;
      const int sx = r % lv.side, sy = r / lv.side;
      return p * lv.npp + lv.off_next + (2 * sx + (k & 1)) + 2 * lv.side * (2 * sy + (k >> 1));
    };
    const long long o = 16LL * ref_pos[i];
    for (int ka = 0; ka < 4; ++ka)
      for (int kb = 0; kb < 4; ++kb) {
        na[o + 4 * ka + kb] = child(a, ka);
        nb[o + 4 * ka + kb] = child(b, kb);
      }
  }
}

// split sorted keys into rows (a) / columns (b)
__global__ void k_split(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ A,
                        int* __restrict__ B) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  A[i] = static_cast<int>(keys[i] >> 32);
  B[i] = static_cast<int>(keys[i] & 0xffffffffu);
}

__device__ __forceinline__ long long lower_bound_key(const unsigned long long* keys, long long n,
                                                     unsigned long long k) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// row starts (nrows + 1) and, when upper != nullptr, the first pair of row t with column > t
__global__ void k_rows(int nrows, const unsigned long long* __restrict__ keys, long long n, int* __restrict__ rs,
                       int* __restrict__ upper) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nrows) return;
  rs[r] = static_cast<int>(lower_bound_key(keys, n, static_cast<unsigned long long>(r) << 32));
  if (upper && r < nrows)
    upper[r] = static_cast<int>(
        lower_bound_key(keys, n, (static_cast<unsigned long long>(r) << 32) | static_cast<unsigned>(r + 1)));
}
// position of the transposed pair; -1 if the relation is not symmetric
__global__ void k_trans(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ trans) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i], t = (k << 32) | (k >> 32);
  const long long j = lower_bound_key(keys, n, t);
  trans[i] = (j < n && keys[j] == t) ? static_cast<int>(j) : -1;
}

unsigned blocks(long long n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

// ---- element boxes, tree boxes, diagonals and near-pair classes on the device.
// Every floating-point step is an explicit round-to-nearest intrinsic in the
// host's (and the reference's) operation order, so the results are bit-identical
// (host code: -ffp-contract=off).
struct PatchDesc {
  int pu, pv, nu, nv;          // degrees, control-point counts
  int ku_off, kv_off, cp_off;  // offsets into knots / control points
};
constexpr int kMaxSetupDeg = 15;

__device__ int find_span_dev(const double* __restrict__ knots, int p, int k, double x) {  // splines.cpp:20-38
  if (x >= knots[k]) {
    int j = k - 1;
    while (knots[j + 1] <= knots[j]) --j;
    return j;
  }
  int lo = p, hi = k;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (x < knots[mid]) hi = mid;
    else lo = mid;
  }
  return lo;
}
__device__ void basis_values_dev(const double* __restrict__ knots, int p, int span, double x, double* out) {  // splines.cpp:69-86
  double left[kMaxSetupDeg + 1], right[kMaxSetupDeg + 1];
  out[0] = 1.0;
  for (int j = 1; j <= p; ++j) {
    left[j] = __dsub_rn(x, knots[span + 1 - j]);
    right[j] = __dsub_rn(knots[span + j], x);
    double saved = 0.0;
    for (int r = 0; r < j; ++r) {
      const double den = __dadd_rn(right[r + 1], left[j - r]);
      const double tmp = den > 0.0 ? __ddiv_rn(out[r], den) : 0.0;
      out[r] = __dadd_rn(saved, __dmul_rn(right[r + 1], tmp));
      saved = __dmul_rn(left[j - r], tmp);
    }
    out[j] = saved;
  }
}
// Discretization::build_elements (spaces.cpp:117-147): box of (degree + 2)^2 surface
// samples (eval_patch, splines.cpp:183-216: the point only), inflated by 1.1
__global__ void k_element_boxes(int ne, int epp, int n1, double h, int ns, const PatchDesc* __restrict__ pd,
                                const double* __restrict__ knots, const double* __restrict__ cw,
                                const double* __restrict__ w, int npp, int leaf_off, DevBox* __restrict__ box) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= ne) return;
  const int p = e / epp, r = e % epp, iy = r / n1, ix = r % n1;
  const PatchDesc D = pd[p];
  const double* ku = knots + D.ku_off;
  const double* kv = knots + D.kv_off;
  const double ox = __dmul_rn(static_cast<double>(ix), h), oy = __dmul_rn(static_cast<double>(iy), h);
  double mn[3] = {1.7976931348623157e308, 1.7976931348623157e308, 1.7976931348623157e308};
  double mx[3] = {-1.7976931348623157e308, -1.7976931348623157e308, -1.7976931348623157e308};
  const double den = static_cast<double>(ns) - 1.0;
  for (int a = 0; a < ns; ++a)
    for (int b = 0; b < ns; ++b) {
      const double u = __dadd_rn(ox, __ddiv_rn(__dmul_rn(h, static_cast<double>(a)), den));
      const double v = __dadd_rn(oy, __ddiv_rn(__dmul_rn(h, static_cast<double>(b)), den));
      double bu[kMaxSetupDeg + 1], bv[kMaxSetupDeg + 1];
      const int su = find_span_dev(ku, D.pu, D.nu, u), sv = find_span_dev(kv, D.pv, D.nv, v);
      basis_values_dev(ku, D.pu, su, u, bu);
      basis_values_dev(kv, D.pv, sv, v, bv);
      const int fu = su - D.pu, fv = sv - D.pv;
      double N[3] = {0.0, 0.0, 0.0}, W = 0.0;
      for (int j = 0; j <= D.pv; ++j)
        for (int i = 0; i <= D.pu; ++i) {
          const int idx = D.cp_off + (fu + i) + (fv + j) * D.nu;
          const double t = __dmul_rn(bu[i], bv[j]);
          for (int k = 0; k < 3; ++k) N[k] = __dadd_rn(N[k], __dmul_rn(cw[3 * idx + k], t));
          W = __dadd_rn(W, __dmul_rn(__dmul_rn(w[idx], bu[i]), bv[j]));
        }
      for (int k = 0; k < 3; ++k) {
        const double x = __ddiv_rn(N[k], W);
        mn[k] = fmin(mn[k], x);
        mx[k] = fmax(mx[k], x);
      }
    }
  DevBox out;
  for (int k = 0; k < 3; ++k) {
    const double c = __ddiv_rn(__dadd_rn(mn[k], mx[k]), 2.0);
    const double half = __dmul_rn(1.1, __dsub_rn(mx[k], c));
    out.mn[k] = __dsub_rn(c, half);
    out.mx[k] = __dadd_rn(c, half);
  }
  box[p * npp + leaf_off + r] = out;  // leaf node of the element
}
// ClusterTree boxes above the leaves (h2.cpp:49-78): union of the four children
__global__ void k_tree_boxes(int np, int level, int npp, int off_l, int off_c, DevBox* __restrict__ box) {
  const int n = 1 << level, per = n * n;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= np * per) return;
  const int p = i / per, r = i % per, sx = r % n, sy = r / n;
  DevBox b;
  for (int k = 0; k < 3; ++k) {
    b.mn[k] = 1.7976931348623157e308;
    b.mx[k] = -1.7976931348623157e308;
  }
  for (int c = 0; c < 4; ++c) {
    const DevBox ch = box[p * npp + off_c + (2 * sx + (c & 1)) + (2 * n) * (2 * sy + (c >> 1))];
    for (int k = 0; k < 3; ++k) {
      b.mn[k] = fmin(b.mn[k], ch.mn[k]);
      b.mx[k] = fmax(b.mx[k], ch.mx[k]);
    }
  }
  box[p * npp + off_l + r] = b;
}
__global__ void k_diag(int nn, const DevBox* __restrict__ box, double* __restrict__ diag) {  // Box::diag_norm
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nn) return;
  const DevBox b = box[i];
  const double a0 = __dsub_rn(b.mx[0], b.mn[0]), a1 = __dsub_rn(b.mx[1], b.mn[1]), a2 = __dsub_rn(b.mx[2], b.mn[2]);
  diag[i] = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(a0, a0), __dmul_rn(a1, a1)), __dmul_rn(a2, a2)));
}

// Discretization::classify_pair (spaces.cpp:309-394) of every near pair (as
// build_plan calls it: on (min, max)); map bits swap | flip_u << 1 | flip_v << 2
__device__ __forceinline__ int map_edge_bits(int edge, int rev) {  // quadrature.cpp:52-63
  switch (edge) {
    case 0: return rev ? 2 : 0;
    case 1: return 1 | 2 | (rev ? 4 : 0);
    case 2: return (rev ? 2 : 0) | 4;
    default: return 1 | (rev ? 4 : 0);
  }
}
__device__ __forceinline__ int map_corner_bits(int corner) {  // quadrature.cpp:65-73
  return ((corner & 1) ? 2 : 0) | ((corner & 2) ? 4 : 0);
}
__device__ __forceinline__ bool on_edge(int edge, int ix, int iy, int n) {
  return edge == 0 ? iy == 0 : edge == 1 ? ix == n - 1 : edge == 2 ? iy == n - 1 : ix == 0;
}
__device__ __forceinline__ bool at_corner(int corner, int ix, int iy, int n) {
  const int cx = (corner == 1 || corner == 3) ? n - 1 : 0, cy = corner >= 2 ? n - 1 : 0;
  return ix == cx && iy == cy;
}
__global__ void k_classify(long long nq, const int* __restrict__ na, const int* __restrict__ nb, int epp, int n, int np,
                           const int* __restrict__ edge_rs, const int* __restrict__ edges,
                           const int* __restrict__ corner_rs, const int* __restrict__ corners,
                           unsigned char* __restrict__ cls, unsigned char* __restrict__ map_a,
                           unsigned char* __restrict__ map_b) {
  const long long q = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (q >= nq) return;
  const int e0 = na[q], e1 = nb[q];
  const int ea = min(e0, e1), eb = max(e0, e1);
  int c = 0, ma = 0, mb = 0;  // kFar
  if (ea == eb) {
    c = 3;  // kCoincident
  } else {
    const int pa = ea / epp, ra = ea % epp, ax = ra % n, ay = ra / n;
    const int pb = eb / epp, rb = eb % epp, bx = rb % n, by = rb / n;
    int best = 0;
    if (pa == pb) {
      const int dx = bx - ax, dy = by - ay;
      if (abs(dx) <= 1 && abs(dy) <= 1) {
        if (abs(dx) + abs(dy) == 1) {
          int edge_a, edge_b;
          if (dx == 1) { edge_a = 1; edge_b = 3; }
          else if (dx == -1) { edge_a = 3; edge_b = 1; }
          else if (dy == 1) { edge_a = 2; edge_b = 0; }
          else { edge_a = 0; edge_b = 2; }
          c = 2;
          ma = map_edge_bits(edge_a, 0);
          mb = map_edge_bits(edge_b, 0);
          best = 2;
        } else {
          const int ca = (dx > 0 ? 1 : 0) + (dy > 0 ? 2 : 0), cb = (dx > 0 ? 0 : 1) + (dy > 0 ? 0 : 2);
          c = 1;
          ma = map_corner_bits(ca);
          mb = map_corner_bits(cb);
          best = 1;
        }
      }
    }
    if (best < 2) {
      for (int i = edge_rs[pa * np + pb]; i < edge_rs[pa * np + pb + 1]; ++i) {
        const int ed_a = edges[3 * i], ed_b = edges[3 * i + 1], rev = edges[3 * i + 2];
        if (!on_edge(ed_a, ax, ay, n) || !on_edge(ed_b, bx, by, n)) continue;
        const int sa = (ed_a == 0 || ed_a == 2) ? ax : ay;
        const int sb_raw = (ed_b == 0 || ed_b == 2) ? bx : by;
        const int sb = rev ? n - 1 - sb_raw : sb_raw;
        if (sa == sb) {
          c = 2;
          ma = map_edge_bits(ed_a, 0);
          mb = map_edge_bits(ed_b, rev);
          best = 2;
          break;
        }
        if (abs(sa - sb) == 1 && best < 1) {
          const int end_a = sb > sa ? 1 : 0, end_b = rev ? end_a : 1 - end_a;
          const int tbl[4][2] = {{0, 1}, {1, 3}, {2, 3}, {0, 2}};  // edge_end_corner
          c = 1;
          ma = map_corner_bits(tbl[ed_a][end_a]);
          mb = map_corner_bits(tbl[ed_b][end_b]);
          best = 1;
        }
      }
    }
    if (best < 1 && pa != pb) {
      for (int i = corner_rs[pa * np + pb]; i < corner_rs[pa * np + pb + 1]; ++i) {
        const int ca = corners[2 * i], cb = corners[2 * i + 1];
        if (at_corner(ca, ax, ay, n) && at_corner(cb, bx, by, n)) {
          c = 1;
          ma = map_corner_bits(ca);
          mb = map_corner_bits(cb);
          best = 1;
          break;
        }
      }
    }
    if (best == 0) { c = 0; ma = 0; mb = 0; }
  }
  cls[q] = static_cast<unsigned char>(c);
  map_a[q] = static_cast<unsigned char>(ma);
  map_b[q] = static_cast<unsigned char>(mb);
}

void device_partition(H2Plan& P, const Discretization& d, double eta, int device) {
  const int L = P.depth, np = P.n_patches, nn = P.n_nodes, ne = d.element_count();
  const int epp = d.elements_per_patch(), n1 = 1 << L;
  IGB_PCUDA(cudaSetDevice(device));
  cudaStream_t st;
  {  // highest priority: the setup kernels run ahead of the singular integrals already queued on the device
    int lo = 0, hi = 0;
    IGB_PCUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    IGB_PCUDA(cudaStreamCreateWithPriority(&st, cudaStreamNonBlocking, hi));
  }
  std::vector<void*> mem;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    IGB_PCUDA(cudaMallocAsync(&p, bytes ? bytes : 8, st));
    mem.push_back(p);
    return p;
  };
  auto release = [&] {
    cudaStreamSynchronize(st);
    for (void* p : mem) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  };
  try {
    // element boxes from the patches, tree boxes and diagonals: all on the device
    const Geometry& G = d.geometry();
    std::vector<PatchDesc> hpd(np);
    std::vector<double> hk, hcw, hw;
    for (int p = 0; p < np; ++p) {
      const Patch& S = G.patch(p);
      if (S.kv_u.degree > kMaxSetupDeg || S.kv_v.degree > kMaxSetupDeg)
        throw std::invalid_argument("B200 H2: device setup supports geometry degrees up to 15");
      hpd[p] = {S.kv_u.degree, S.kv_v.degree, S.count_u(), S.count_v(), static_cast<int>(hk.size()),
                static_cast<int>(hk.size() + S.kv_u.knots.size()), static_cast<int>(hw.size())};
      hk.insert(hk.end(), S.kv_u.knots.begin(), S.kv_u.knots.end());
      hk.insert(hk.end(), S.kv_v.knots.begin(), S.kv_v.knots.end());
      hcw.insert(hcw.end(), S.cw.begin(), S.cw.end());
      hw.insert(hw.end(), S.w.begin(), S.w.end());
    }
    auto up = [&](const void* src, size_t bytes) {
      void* p = alloc(bytes);
      if (bytes) IGB_PCUDA(cudaMemcpyAsync(p, src, bytes, cudaMemcpyHostToDevice, st));
      return p;
    };
    const PatchDesc* dpd = static_cast<const PatchDesc*>(up(hpd.data(), hpd.size() * sizeof(PatchDesc)));
    const double* dk = static_cast<const double*>(up(hk.data(), hk.size() * 8));
    const double* dcw = static_cast<const double*>(up(hcw.data(), hcw.size() * 8));
    const double* dw = static_cast<const double*>(up(hw.data(), hw.size() * 8));
    DevBox* dbox = static_cast<DevBox*>(alloc(nn * sizeof(DevBox)));
    double* ddiag = static_cast<double*>(alloc(nn * sizeof(double)));
    k_element_boxes<<<blocks(ne), 256, 0, st>>>(ne, epp, n1, 1.0 / n1, d.degree() + 2, dpd, dk, dcw, dw, P.npp,
                                                P.level_offset[L], dbox);
    for (int l = L - 1; l >= 0; --l)
      k_tree_boxes<<<blocks(static_cast<long long>(np) << (2 * l)), 256, 0, st>>>(np, l, P.npp, P.level_offset[l],
                                                                                  P.level_offset[l + 1], dbox);
    k_diag<<<blocks(nn), 256, 0, st>>>(nn, dbox, ddiag);
    IGB_PCUDA(cudaGetLastError());
    {
      std::vector<DevBox> hb(nn);
      IGB_PCUDA(cudaMemcpyAsync(hb.data(), dbox, nn * sizeof(DevBox), cudaMemcpyDeviceToHost, st));
      IGB_PCUDA(cudaStreamSynchronize(st));
      for (int i = 0; i < nn; ++i)
        for (int k = 0; k < 3; ++k) {
          P.node_box[i].mn[k] = hb[i].mn[k];
          P.node_box[i].mx[k] = hb[i].mx[k];
        }
    }
    // level-0 frontier: every ordered root pair
    std::vector<int> ha, hbv;
    for (int a = 0; a < np; ++a)
      for (int b = 0; b < np; ++b) {
        ha.push_back(static_cast<int>(P.node_id(a, 0, 0, 0)));
        hbv.push_back(static_cast<int>(P.node_id(b, 0, 0, 0)));
      }
    long long n = static_cast<long long>(ha.size());
    int* fa = static_cast<int*>(alloc(n * sizeof(int)));
    int* fb = static_cast<int*>(alloc(n * sizeof(int)));
    IGB_PCUDA(cudaMemcpyAsync(fa, ha.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    IGB_PCUDA(cudaMemcpyAsync(fb, hbv.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    std::vector<unsigned long long*> far_chunks;
    std::vector<long long> far_counts;
    unsigned long long* near_keys = nullptr;
    long long n_near = 0;
    for (int l = 0; l <= L && n > 0; ++l) {
      unsigned char* dec = static_cast<unsigned char*>(alloc(n));
      int* flags = static_cast<int*>(alloc(3 * n * sizeof(int)));
      int* pos = static_cast<int*>(alloc(3 * (n + 1) * sizeof(int)));
      k_decide<<<blocks(n), 256, 0, st>>>(n, fa, fb, dbox, ddiag, eta, l == L, dec, flags, flags + n, flags + 2 * n);
      IGB_PCUDA(cudaGetLastError());
      size_t tmp_bytes = 0;
      IGB_PCUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, pos, static_cast<int>(n), st));
      void* tmp = alloc(tmp_bytes);
      int cnt[3];
      for (int k = 0; k < 3; ++k) {  // exclusive scans; count = last position + last flag
        IGB_PCUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags + k * n, pos + k * (n + 1), static_cast<int>(n), st));
        int last_pos = 0, last_flag = 0;
        IGB_PCUDA(cudaMemcpyAsync(&last_pos, pos + k * (n + 1) + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        IGB_PCUDA(cudaMemcpyAsync(&last_flag, flags + k * n + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        IGB_PCUDA(cudaStreamSynchronize(st));
        cnt[k] = last_pos + last_flag;
      }
      unsigned long long* fk = static_cast<unsigned long long*>(alloc(std::max(1, cnt[0]) * sizeof(unsigned long long)));
      if (cnt[1] > 0) near_keys = static_cast<unsigned long long*>(alloc(cnt[1] * sizeof(unsigned long long)));
      const long long nnext = 16LL * cnt[2];
      if (nnext > 0x7fffffffLL) throw std::runtime_error("B200 H2: too many block pairs for 32-bit indexing");
      int* na = static_cast<int*>(alloc(std::max<long long>(1, nnext) * sizeof(int)));
      int* nb = static_cast<int*>(alloc(std::max<long long>(1, nnext) * sizeof(int)));
      Level lv{P.npp, P.level_offset[l], l < L ? P.level_offset[l + 1] : 0, 1 << l};
      k_emit<<<blocks(n), 256, 0, st>>>(n, fa, fb, dec, pos, pos + (n + 1), pos + 2 * (n + 1), lv, epp, n1, fk, 0,
                                        near_keys, na, nb);
      IGB_PCUDA(cudaGetLastError());
      far_chunks.push_back(fk);
      far_counts.push_back(cnt[0]);
      if (cnt[1] > 0) n_near = cnt[1];
      fa = na;
      fb = nb;
      n = nnext;
    }
    // concatenate and sort the far keys; sort the near keys
    long long n_far = 0;
    for (long long c : far_counts) n_far += c;
    if (n_far > 0x7fffffffLL || n_near > 0x7fffffffLL)
      throw std::runtime_error("B200 H2: too many block pairs for 32-bit indexing");
    auto sort_keys = [&](unsigned long long* in, long long cnt) {
      unsigned long long* out = static_cast<unsigned long long*>(alloc(std::max<long long>(1, cnt) * 8));
      size_t tb = 0;
      IGB_PCUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, static_cast<int>(cnt), 0, 64, st));
      void* t = alloc(tb);
      IGB_PCUDA(cub::DeviceRadixSort::SortKeys(t, tb, in, out, static_cast<int>(cnt), 0, 64, st));
      return out;
    };
    unsigned long long* fall = static_cast<unsigned long long*>(alloc(std::max<long long>(1, n_far) * 8));
    {
      long long o = 0;
      for (size_t i = 0; i < far_chunks.size(); ++i) {
        if (far_counts[i])
          IGB_PCUDA(cudaMemcpyAsync(fall + o, far_chunks[i], far_counts[i] * 8, cudaMemcpyDeviceToDevice, st));
        o += far_counts[i];
      }
    }
    unsigned long long* fsorted = sort_keys(fall, n_far);
    unsigned long long* nsorted = n_near ? sort_keys(near_keys, n_near) : nullptr;
    // rows, columns, row starts, upper starts, transposes
    int* dfa = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dfb = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dtr = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dfrs = static_cast<int*>(alloc((nn + 1) * 4));
    int* dup = static_cast<int*>(alloc(nn * 4));
    int* dna = static_cast<int*>(alloc(std::max<long long>(1, n_near) * 4));
    int* dnb = static_cast<int*>(alloc(std::max<long long>(1, n_near) * 4));
    int* dnrs = static_cast<int*>(alloc((ne + 1) * 4));
    if (n_far) {
      k_split<<<blocks(n_far), 256, 0, st>>>(n_far, fsorted, dfa, dfb);
      k_trans<<<blocks(n_far), 256, 0, st>>>(n_far, fsorted, dtr);
    }
    k_rows<<<blocks(nn + 1), 256, 0, st>>>(nn, fsorted, n_far, dfrs, dup);
    if (n_near) k_split<<<blocks(n_near), 256, 0, st>>>(n_near, nsorted, dna, dnb);
    k_rows<<<blocks(ne + 1), 256, 0, st>>>(ne, nsorted, n_near, dnrs, nullptr);
    IGB_PCUDA(cudaGetLastError());
    // classes and maps of the near pairs
    unsigned char* dcls = static_cast<unsigned char*>(alloc(std::max<long long>(1, 3 * n_near)));
    if (n_near) {
      std::vector<int> ers, eds, crs, cns;
      d.flatten_topology(ers, eds, crs, cns);
      const int* d_ers = static_cast<const int*>(up(ers.data(), ers.size() * 4));
      const int* d_eds = static_cast<const int*>(up(eds.data(), eds.size() * 4));
      const int* d_crs = static_cast<const int*>(up(crs.data(), crs.size() * 4));
      const int* d_cns = static_cast<const int*>(up(cns.data(), cns.size() * 4));
      k_classify<<<blocks(n_near), 256, 0, st>>>(n_near, dna, dnb, epp, n1, np, d_ers, d_eds, d_crs, d_cns, dcls,
                                                 dcls + n_near, dcls + 2 * n_near);
      IGB_PCUDA(cudaGetLastError());
      IGB_PCUDA(cudaStreamSynchronize(st));  // the topology vectors leave scope
    }
    P.near_cls.resize(n_near);
    P.dev_map_a.resize(n_near);
    P.dev_map_b.resize(n_near);
    if (n_near) {
      IGB_PCUDA(cudaMemcpyAsync(P.near_cls.data(), dcls, n_near, cudaMemcpyDeviceToHost, st));
      IGB_PCUDA(cudaMemcpyAsync(P.dev_map_a.data(), dcls + n_near, n_near, cudaMemcpyDeviceToHost, st));
      IGB_PCUDA(cudaMemcpyAsync(P.dev_map_b.data(), dcls + 2 * n_near, n_near, cudaMemcpyDeviceToHost, st));
    }
    P.far_a.resize(n_far);
    P.far_b.resize(n_far);
    P.far_trans.resize(n_far);
    P.far_row_start.resize(nn + 1);
    P.far_upper_start.resize(nn);
    P.near_a.resize(n_near);
    P.near_b.resize(n_near);
    P.near_row_start.resize(ne + 1);
    auto down = [&](std::vector<int>& v, const int* src) {
      if (!v.empty()) IGB_PCUDA(cudaMemcpyAsync(v.data(), src, v.size() * 4, cudaMemcpyDeviceToHost, st));
    };
    down(P.far_a, dfa);
    down(P.far_b, dfb);
    down(P.far_trans, dtr);
    down(P.far_row_start, dfrs);
    down(P.far_upper_start, dup);
    down(P.near_a, dna);
    down(P.near_b, dnb);
    down(P.near_row_start, dnrs);
    IGB_PCUDA(cudaStreamSynchronize(st));
  } catch (...) {
    release();
    throw;
  }
  release();
  for (int t : P.far_trans)
    if (t < 0) throw std::logic_error("B200 H2: admissible relation is not symmetric");
}

}  // namespace igb
