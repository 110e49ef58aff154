// B200 (sm_100a) kernels for the H² single-layer / EFIE operator:
//   assembly  : element quadrature caches + Chebyshev moments (h2.cpp:131-173,
//               pair_integration.hpp:40-73), interpolation-node images
//               (h2.cpp:182-196), far couplings (h2.cpp:218-229), regular near
//               blocks (pair_integration.hpp:76-95) and Sauter-Schwab singular
//               blocks batched by class (pair_integration.hpp:98-148,
//               quadrature.cpp:82-199);
//   matvec    : the seven phases of H2Matrix::apply (h2.cpp:254-378).
// All FP64.  Every reduction is a fixed-order loop (no atomics), so results
// are bitwise reproducible run to run.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>

#include "igb_device.hpp"

#include "igb_common.cuh"

namespace igb {
namespace dev {

// ------------------------------------------------------ device args
struct GeoArgs {
  const double* cells;   // [cell][kCellStride]
  const int* el_cell;
  const double* tab_a;
  const double* tab_b;
  int level, epp;
  double h;
  KParams kp;
};

// offset (in scalars) of entry (la, lb) of near slot q in the row layout
__device__ __forceinline__ size_t near_off(const int* __restrict__ near_a, const int* __restrict__ near_rs, int q,
                                           int la, int lb, int NL) {
  const int e = near_a[q];
  const int rs = near_rs[e];
  const int cnt = near_rs[e + 1] - rs;
  return static_cast<size_t>(rs) * NL * NL + (static_cast<size_t>(la) * cnt + (q - rs)) * NL + lb;
}

// ---------------------------------------------------- K1: element caches
// Per element: quadrature points, weighted shapes (far caches,
// pair_integration.hpp:40-73) and Chebyshev moments (h2.cpp:131-173).
template <class KT>
__global__ void __launch_bounds__(128) k_element(GeoArgs g, int nf, const double* __restrict__ gx,
                                                 const double* __restrict__ gw, int m,
                                                 const double* __restrict__ lag,  // [m][nf]
                                                 double* __restrict__ cpts, double* __restrict__ cval,
                                                 double* __restrict__ mom) {
  constexpr int NL = KT::NL, NC = KT::NC;
  extern __shared__ __align__(16) double sm[];
  double* cf = sm;
  double* tab = sm + 104;
  double* wphi = tab + KT::TABN;  // [nq][NC*NL]
  const int e = blockIdx.x, tid = threadIdx.x;
  const int cell = g.el_cell[e];
  const int r = e % g.epp, n1 = 1 << g.level, ix = r % n1, iy = r / n1;
  for (int i = tid; i < 100; i += blockDim.x) cf[i] = g.cells[static_cast<size_t>(cell) * kCellStride + i];
  load_tables<KT>(tab, g.tab_a, g.tab_b, ix, iy, tid, blockDim.x);
  __syncthreads();
  const double u0 = g.cells[static_cast<size_t>(cell) * kCellStride + 100];
  const double v0 = g.cells[static_cast<size_t>(cell) * kCellStride + 101];
  const double ox = ix * g.h, oy = iy * g.h;
  const int nq = nf * nf;
  for (int q = tid; q < nq; q += blockDim.x) {
    const int a = q % nf, b = q / nf;
    const double ul = gx[a], vl = gx[b];
    double x[3], du[3], dv[3];
    jet<4>(cf, ox + g.h * ul - u0, oy + g.h * vl - v0, x, du, dv);
    const double sg = sqrt_g_of(du, dv);
    const double w = gw[a] * gw[b] * sg * g.h * g.h;
    double sh[NC][NL];
    shapes<KT>(tab, ul, vl, g.h, du, dv, sg, sh);
    for (int k = 0; k < 3; ++k) cpts[(static_cast<size_t>(e) * nq + q) * 3 + k] = x[k];
#pragma unroll
    for (int c = 0; c < NC; ++c)
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        const double v = w * sh[c][l];
        cval[((static_cast<size_t>(e) * NC + c) * nq + q) * NL + l] = v;
        wphi[q * (NC * NL) + c * NL + l] = v;
      }
  }
  __syncthreads();
  const int mm = m * m, rows = NC * mm;
  for (int o = tid; o < NL * rows; o += blockDim.x) {
    const int l = o / rows, rr = o % rows, c = rr / mm, nu = rr % mm, iu = nu % m, iv = nu / m;
    double acc = 0.0;
    for (int b = 0; b < nf; ++b) {
      double in = 0.0;
      for (int a = 0; a < nf; ++a) in = fma(lag[iu * nf + a], wphi[(a + nf * b) * (NC * NL) + c * NL + l], in);
      acc = fma(lag[iv * nf + b], in, acc);
    }
    mom[(static_cast<size_t>(e) * NL + l) * rows + rr] = acc;
  }
}

// --------------------------------------------------------- K2: images
struct PatchDev {
  const int* info;      // per patch: cell_base, pu, pv, nku, nkv, ku_off, kv_off
  const double* knots;
};
__device__ __forceinline__ int find_span_dev(const double* k, int p, int nk, double x) {  // splines.cpp:20-38
  const int n = nk - p - 1;
  if (x >= k[n]) {
    int j = n - 1;
    while (k[j + 1] <= k[j]) --j;
    return j;
  }
  int lo = p, hi = n;
  while (hi - lo > 1) {
    const int mid = (lo + hi) / 2;
    if (x < k[mid]) hi = mid;
    else lo = mid;
  }
  return lo;
}
__global__ void k_images(int n_nodes, int m, const double* __restrict__ cheb, const int* __restrict__ node_patch,
                         const int* __restrict__ node_level, const int* __restrict__ node_sx,
                         const int* __restrict__ node_sy, PatchDev pd, const double* __restrict__ cells,
                         double* __restrict__ img) {
  const int mm = m * m;
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_nodes) * mm) return;
  const int node = static_cast<int>(idx / mm), nu = static_cast<int>(idx % mm), iu = nu % m, iv = nu / m;
  const int p = node_patch[node];
  const double hs = 1.0 / (1 << node_level[node]);
  const double u = hs * (node_sx[node] + cheb[iu]);
  const double v = hs * (node_sy[node] + cheb[iv]);
  const int* inf = pd.info + 7 * p;
  const int su = find_span_dev(pd.knots + inf[5], inf[1], inf[3], u);
  const int sv = find_span_dev(pd.knots + inf[6], inf[2], inf[4], v);
  const int nsv = (inf[4] - inf[2] - 1) - inf[2];
  const int cell = inf[0] + (su - inf[1]) * nsv + (sv - inf[2]);
  const double* cf = cells + static_cast<size_t>(cell) * kCellStride;
  double x[3];
  point_only<4>(cf, u - cf[100], v - cf[101], x);
  for (int k = 0; k < 3; ++k) img[idx * 3 + k] = x[k];
}

// ------------------------------------------------------ K3: couplings
// K[q][mu][nu] = G(|img_ta[nu] - img_tb[mu]|)  (h2.cpp:218-229)
template <class KT>
__global__ void __launch_bounds__(256) k_couplings(long long n_pairs, int mm, const int* __restrict__ far_a,
                                                   const int* __restrict__ far_b, const double* __restrict__ img,
                                                   KParams kp, double* __restrict__ out) {
  using S = typename KT::S;
  S* K = reinterpret_cast<S*>(out);
  const long long mm2 = static_cast<long long>(mm) * mm;
  const long long total = n_pairs * mm2;
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long q = i / mm2;
    const int r = static_cast<int>(i % mm2), nu = r % mm, mu = r / mm;
    const double* a = img + (static_cast<size_t>(far_a[q]) * mm + nu) * 3;
    const double* b = img + (static_cast<size_t>(far_b[q]) * mm + mu) * 3;
    const double d0 = a[0] - b[0], d1 = a[1] - b[1], d2 = a[2] - b[2];
    K[i] = green_k<KT>(d0 * d0 + d1 * d1 + d2 * d2, kp);
  }
}

// --------------------------------------------------- K4: regular near
// blk = sum_c w_c A_c^T (K B_c)  (pair_integration.hpp:76-95)
// Regular blocks (pair_integration.hpp far_block 76-95): tensor Gauss on both
// elements from the element caches, np pairs per CTA (one work item per
// thread).  pair(p, ea, eb) names pair p; put(p, la, lb, v) stores entry
// (la, lb) of its block.
template <class KT, class PairFn, class PutFn>
__device__ __forceinline__ void regular_body(int np, int nq, const double* __restrict__ cpts,
                                             const double* __restrict__ cval, KParams kp, PairFn pair, PutFn put) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NC = KT::NC;
  extern __shared__ __align__(16) double sm[];
  S* KB = reinterpret_cast<S*>(sm);  // [np][NC][nq][NL]
  for (int it = threadIdx.x; it < np * NC * nq; it += blockDim.x) {
    const int p = it / (NC * nq), r = it % (NC * nq), c = r / nq, i = r % nq;
    int ea, eb;
    pair(p, ea, eb);
    const double* pa = cpts + static_cast<size_t>(ea) * nq * 3;
    const double* pb = cpts + static_cast<size_t>(eb) * nq * 3;
    const double xa = pa[3 * i], ya = pa[3 * i + 1], za = pa[3 * i + 2];
    const double* B = cval + (static_cast<size_t>(eb) * NC + c) * nq * NL;
    S acc[NL];
#pragma unroll
    for (int l = 0; l < NL; ++l) acc[l] = zero<S>();
    for (int j = 0; j < nq; ++j) {
      const double d0 = xa - pb[3 * j], d1 = ya - pb[3 * j + 1], d2 = za - pb[3 * j + 2];
      const S gk = green_k<KT>(d0 * d0 + d1 * d1 + d2 * d2, kp);
#pragma unroll
      for (int l = 0; l < NL; ++l) fmac(acc[l], gk, B[j * NL + l]);
    }
#pragma unroll
    for (int l = 0; l < NL; ++l) KB[((p * NC + c) * nq + i) * NL + l] = acc[l];
  }
  __syncthreads();
  for (int o = threadIdx.x; o < np * NL * NL; o += blockDim.x) {
    const int p = o / (NL * NL), la = (o / NL) % NL, lb = o % NL;
    int ea, eb;
    pair(p, ea, eb);
    S tot = zero<S>();
#pragma unroll
    for (int c = 0; c < NC; ++c) {
      const double* A = cval + (static_cast<size_t>(ea) * NC + c) * nq * NL;
      S s = zero<S>();
      for (int i = 0; i < nq; ++i) fmac(s, KB[((p * NC + c) * nq + i) * NL + lb], A[i * NL + la]);
      if constexpr (KT::KIND == 2) {
        if (c == 3) s = s * mk(kp.dwx, kp.dwy);
      }
      tot = tot + s;
    }
    put(p, la, lb, tot);
  }
}

// Regular near blocks of the H2 near field: P unique pairs (ea < eb) per CTA;
// the block goes to the slot of (ea, eb) and its transpose to the slot of
// (eb, ea) (either may be another rank's, -1).
template <class KT>
__global__ void __launch_bounds__(128) k_regular(int n_pairs, int P, const int* __restrict__ slot_ab,
                                                 const int* __restrict__ slot_ba, const int* __restrict__ near_a,
                                                 const int* __restrict__ near_b, const int* __restrict__ near_rs,
                                                 const int* __restrict__ near_ea, int nq,
                                                 const double* __restrict__ cpts, const double* __restrict__ cval,
                                                 KParams kp, double* __restrict__ near) {
  using S = typename KT::S;
  constexpr int NL = KT::NL;
  const int p0 = blockIdx.x * P, np = min(P, n_pairs - p0);
  S* out = reinterpret_cast<S*>(near);
  regular_body<KT>(
      np, nq, cpts, cval, kp,
      [&](int p, int& ea, int& eb) {
        const int qab = slot_ab[p0 + p];
        if (qab >= 0) {
          ea = near_ea[qab];
          eb = near_b[qab];
        } else {
          const int qba = slot_ba[p0 + p];
          ea = near_b[qba];
          eb = near_ea[qba];
        }
      },
      [&](int p, int la, int lb, S v) {
        const int qab = slot_ab[p0 + p], qba = slot_ba[p0 + p];
        if (qab >= 0) out[near_off(near_a, near_rs, qab, la, lb, NL)] = v;
        if (qba >= 0) out[near_off(near_a, near_rs, qba, lb, la, NL)] = v;
      });
}

// ---- dense Galerkin matrix (assembly.cpp:16-53)
// all pairs (ea, eb), ea in [ea0, ea0 + nrow): regular blocks into the chunk
// buffer buf[(ea - ea0) * ne + eb][la][lb] (singular pairs overwritten next)
template <class KT>
__global__ void __launch_bounds__(128) k_regular_dense(long long n_pairs, int P, int ea0, int ne, int nq,
                                                       const double* __restrict__ cpts,
                                                       const double* __restrict__ cval, KParams kp,
                                                       double* __restrict__ buf) {
  using S = typename KT::S;
  constexpr int NL = KT::NL;
  const long long p0 = static_cast<long long>(blockIdx.x) * P;
  const int np = static_cast<int>(min(static_cast<long long>(P), n_pairs - p0));
  S* out = reinterpret_cast<S*>(buf);
  regular_body<KT>(
      np, nq, cpts, cval, kp,
      [&](int p, int& ea, int& eb) {
        const long long g = p0 + p;
        ea = ea0 + static_cast<int>(g / ne);
        eb = static_cast<int>(g % ne);
      },
      [&](int p, int la, int lb, S v) { out[((p0 + p) * NL + la) * NL + lb] = v; });
}
// singular blocks (compact, ea <= eb) of the pairs with a row in the chunk;
// ea > eb rows get the transpose (pair_integration.hpp:139-148)
template <class S, int NL>
__global__ void k_dense_sing_place(int n_items, const int* __restrict__ ea, const int* __restrict__ eb,
                                   const S* __restrict__ blk, int ea0, int nrow, int ne, S* __restrict__ buf) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_items) * NL * NL) return;
  const int k = static_cast<int>(idx / (NL * NL)), o = static_cast<int>(idx % (NL * NL)), la = o / NL, lb = o % NL;
  const int a = ea[k], b = eb[k];
  const S v = blk[idx];
  if (a >= ea0 && a < ea0 + nrow) buf[((static_cast<size_t>(a - ea0) * ne + b) * NL + la) * NL + lb] = v;
  if (a != b && b >= ea0 && b < ea0 + nrow) buf[((static_cast<size_t>(b - ea0) * ne + a) * NL + lb) * NL + la] = v;
}
// row strips: strip[(ea - ea0) nl + la][j] = sum over the incidences (eb, lb)
// of DOF j in ascending (eb, lb) of sign * block(ea, eb)[la][lb]
template <class S, int NL>
__global__ void k_dense_strip(int nrow, int nd, int ne, const int* __restrict__ dof_start,
                              const int* __restrict__ dof_inc, const double* __restrict__ sg,
                              const S* __restrict__ buf, S* __restrict__ strip) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(nrow) * NL * nd) return;
  const int j = static_cast<int>(idx % nd), r = static_cast<int>(idx / nd), el = r / NL, la = r % NL;
  S acc = zero<S>();
  for (int i = dof_start[j]; i < dof_start[j + 1]; ++i) {
    const int k = dof_inc[i], eb = k / NL, lb = k % NL;
    acc = acc + buf[((static_cast<size_t>(el) * ne + eb) * NL + la) * NL + lb] * sg[k];
  }
  strip[idx] = acc;
}
// a(i, j) += sign * strip row of every incidence (ea, la) of DOF i inside the
// chunk, ascending ea (column-major a; the reference's fixed-order reduction)
template <class S, int NL>
__global__ void k_dense_rows(int n_rows, const int* __restrict__ rows, int nd, const int* __restrict__ dof_start,
                             const int* __restrict__ dof_inc, const double* __restrict__ sg, int ea0, int nrow,
                             const S* __restrict__ strip, S* __restrict__ A) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_rows) * nd) return;
  const int j = static_cast<int>(idx % nd), i = rows[idx / nd];
  S acc = A[static_cast<size_t>(j) * nd + i];
  for (int q = dof_start[i]; q < dof_start[i + 1]; ++q) {
    const int k = dof_inc[q], ea = k / NL;
    if (ea < ea0 || ea >= ea0 + nrow) continue;
    acc = acc + strip[static_cast<size_t>((ea - ea0) * NL + k % NL) * nd + j] * sg[k];
  }
  A[static_cast<size_t>(j) * nd + i] = acc;
}

// ---------------------------------------------------- K5: singular near
// Regularised relative-coordinate rules generated in-register
// (quadrature.cpp:82-177) line by line (rule_line); one CTA per unique pair
// (ea <= eb) writing the compact block, which k_sing_scatter places in the
// two ordered slots (pair_integration.hpp:139-148).

// Sum-factorised geometry jet.  Setup (once per rule line, element, homogeneous
// component): with the fixed cell coordinate f, A_o = sum_k c[o][k] f^k and
// B_o its derivative in f (the inner Horner loops of jet<4>); for a moving v
// the coefficients are read as c[j][i] (o = j), for a moving u as c[i][j].
__device__ __forceinline__ void jet_setup_regs(const double* __restrict__ comp, int v_moves, double f,
                                               double res[10]) {
  const int so = v_moves ? 5 : 1, sk = v_moves ? 1 : 5;
#pragma unroll
  for (int o = 0; o <= kMaxGeomDeg; ++o) {
    double r = comp[o * so + kMaxGeomDeg * sk], rp = 0.0;
#pragma unroll
    for (int k = kMaxGeomDeg - 1; k >= 0; --k) {
      rp = fma(rp, f, r);
      r = fma(r, f, comp[o * so + k * sk]);
    }
    res[o] = r;
    res[5 + o] = rp;
  }
}
__device__ __forceinline__ void jet_setup(const double* __restrict__ comp, int v_moves, double f,
                                          double* __restrict__ out) {
  double res[10];
  jet_setup_regs(comp, v_moves, f, res);
  double2* o2 = reinterpret_cast<double2*>(out);
#pragma unroll
  for (int k = 0; k < 5; ++k) o2[k] = make_double2(res[2 * k], res[2 * k + 1]);
}
// One homogeneous component at the moving coordinate y: the outer Horner loop
// of jet<4> (the same arithmetic when v moves) -> value and the two partials.
__device__ __forceinline__ void jet_comp(const double A[10], int v_moves, double y, double& N, double& Ns,
                                         double& Nt) {
  double n = 0.0, ny = 0.0, nx = 0.0;
#pragma unroll
  for (int o = kMaxGeomDeg; o >= 0; --o) {
    ny = fma(ny, y, n);
    n = fma(n, y, A[o]);
    nx = fma(nx, y, A[5 + o]);
  }
  N = n;
  Ns = v_moves ? nx : ny;
  Nt = v_moves ? ny : nx;
}
// rational quotient of the homogeneous jet (splines.cpp:183-216)
__device__ __forceinline__ void jet_quot(const double N[4], const double Ns[4], const double Nt[4], double x[3],
                                         double du[3], double dv[3]) {
  const double iw = 1.0 / N[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    x[k] = N[k] * iw;
    du[k] = (Ns[k] - x[k] * Ns[3]) * iw;
    dv[k] = (Nt[k] - x[k] * Nt[3]) * iw;
  }
}
// Point of a line from its setup at the moving coordinate y.
__device__ __forceinline__ void jet_line(const double* __restrict__ st, int v_moves, double y, double x[3],
                                         double du[3], double dv[3]) {
  double N[4], Ns[4], Nt[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    // 16 B shared loads (st is 16 B aligned): half the load instructions
    double A[10];
    const double2* A2 = reinterpret_cast<const double2*>(st + c * 10);
#pragma unroll
    for (int k = 0; k < 5; ++k) {
      const double2 v = A2[k];
      A[2 * k] = v.x;
      A[2 * k + 1] = v.y;
    }
    jet_comp(A, v_moves, y, N[c], Ns[c], Nt[c]);
  }
  jet_quot(N, Ns, Nt, x, du, dv);
}
// Vertex lines fix both parameters of element a: its setup tasks finish the
// component's jet at the fixed point ([N, Ns, Nt, -] per component) and the
// points only form the quotient.
__device__ __forceinline__ void jet_fixed(const double* __restrict__ st, double x[3], double du[3], double dv[3]) {
  double N[4], Ns[4], Nt[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double2* A2 = reinterpret_cast<const double2*>(st + c * 10);
    const double2 a = A2[0], b = A2[1];
    N[c] = a.x;
    Ns[c] = a.y;
    Nt[c] = b.x;
  }
  jet_quot(N, Ns, Nt, x, du, dv);
}

// FP64 tensor-core MMA (DMMA, mma.sync m8n8k4): d += a b, one A element
// (row lane/4, column lane%4), one B element (row lane%4, column lane/4) and two
// accumulators (row lane/4, columns 2 (lane%4) + {0, 1}) per lane
// point stride of the DMMA staging [l][point] (== 4 mod 16: the fragment loads of
// a half warp hit 16 distinct bank pairs)
constexpr int kDmmaPstr = 132;
__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// Exact small-integer division by the (runtime) rule order n: float
// reciprocal estimate, then one correction step either way (x < 2^24).
__device__ __forceinline__ int div_n(int x, int n, float rn) {
  int q = __float2int_rz(__int2float_rn(x) * rn);
  q += (q + 1) * n <= x;
  q -= q * n > x;
  return q;
}

// One rule line (fixed sector, i1, i2, i3; i4 runs): after the element maps,
// every coordinate is affine in gx[i4] -- (ua, va, ub, vb) = c0 + c1 gx[i4] --
// and the weight is wl * gw[i4] (the rules of quadrature.cpp:82-177 with the
// maps of quadrature.hpp:25-29 folded in).
template <int CLS>
__device__ __forceinline__ void rule_line(int line, int n, float rn, const double* gx, const double* gw, int ma,
                                          int mb, double c0[4], double c1[4], double& wl, bool half = false) {
  int q = div_n(line, n, rn);
  const int i3 = line - q * n;
  int r = q;
  q = div_n(r, n, rn);
  const int i2 = r - q * n;
  r = q;
  q = div_n(r, n, rn);
  const int i1 = r - q * n;
  const int sec = q;
  const double w3 = gw[i1] * gw[i2] * gw[i3];
  if constexpr (CLS == 3) {  // coincident (quadrature.cpp:82-111)
    // half rule: only the dir = +1 sectors {0, 1, 4, 5}; (dir, sgn) -> (-dir,
    // -sgn) maps z -> -z and swaps the two points with the same weight, so
    // the other four sectors contribute the transpose (added at the end)
    const int sec_ = half ? (((sec >> 1) << 2) | (sec & 1)) : sec;
    const int axis = sec_ >> 2;
    const double dir = (sec_ & 2) ? -1.0 : 1.0, sgn = (sec_ & 1) ? -1.0 : 1.0;
    const double t = gx[i1], s = gx[i2];
    double z1, z2;
    if (axis == 0) {
      z1 = dir * t;
      z2 = sgn * t * s;
    } else {
      z1 = sgn * t * s;
      z2 = dir * t;
    }
    const double lx = 1.0 - fabs(z1), ly = 1.0 - fabs(z2);
    const double x1 = fmax(0.0, -z1) + lx * gx[i3];
    const double x2 = fmax(0.0, -z2);
    c0[0] = x1;      c1[0] = 0.0;
    c0[1] = x2;      c1[1] = ly;
    c0[2] = x1 + z1; c1[2] = 0.0;
    c0[3] = x2 + z2; c1[3] = ly;
    wl = w3 * t * lx * ly;
  } else if constexpr (CLS == 2) {  // edge (quadrature.cpp:113-149)
    const int kind = sec >> 1;
    const double sgn = (sec & 1) ? -1.0 : 1.0;
    // lines run over i3 (the decoded innermost index is i4): the element whose
    // point does not depend on i3 (a for kinds 0 and 2, b for kind 1) is fixed
    // along the line, the other moves its v (t * gx[i3])
    const double t = gx[i1], a = gx[i2], g4 = gx[i3];
    double d, jac;
    if (kind == 2) {
      d = sgn * t;
      jac = t * t * (1.0 - t);
    } else {
      d = sgn * t * a;
      jac = t * t * (1.0 - t * a);
    }
    const double u0 = fmax(0.0, -d), ul = 1.0 - fabs(d);
    c0[0] = fma(ul, g4, u0);     c1[0] = 0.0;
    c0[2] = fma(ul, g4, u0 + d); c1[2] = 0.0;
    if (kind == 0) {
      c0[1] = t;     c1[1] = 0.0;
      c0[3] = 0.0;   c1[3] = t;
    } else if (kind == 1) {
      c0[1] = 0.0;   c1[1] = t;
      c0[3] = t;     c1[3] = 0.0;
    } else {
      c0[1] = t * a; c1[1] = 0.0;
      c0[3] = 0.0;   c1[3] = t;
    }
    wl = w3 * jac;
    (void)i1;
  } else {  // vertex (quadrature.cpp:151-177)
    const double t = gx[i1];
    const double v1 = t * gx[i2], v2 = t * gx[i3];
    for (int k = 0; k < 4; ++k) c1[k] = 0.0;
    switch (sec) {
      case 0: c0[0] = t;  c0[1] = v1; c0[2] = v2; c0[3] = 0.0; c1[3] = t; break;
      case 1: c0[0] = v1; c0[1] = t;  c0[2] = v2; c0[3] = 0.0; c1[3] = t; break;
      case 2: c0[0] = v1; c0[1] = v2; c0[2] = t;  c0[3] = 0.0; c1[3] = t; break;
      default: c0[0] = v1; c0[1] = v2; c0[2] = 0.0; c1[2] = t; c0[3] = t; break;
    }
    wl = w3 * t * t * t;
  }
  // element maps on the affine forms: swap u/v, then reflect u and/or v
  auto map2 = [](int bits, double& a0, double& a1, double& b0, double& b1) {
    if (bits & 1) {
      double t0 = a0, t1 = a1;
      a0 = b0; a1 = b1; b0 = t0; b1 = t1;
    }
    if (bits & 2) { a0 = 1.0 - a0; a1 = -a1; }
    if (bits & 4) { b0 = 1.0 - b0; b1 = -b1; }
  };
  map2(ma, c0[0], c1[0], c0[1], c1[1]);
  map2(mb, c0[2], c1[2], c0[3], c1[3]);
}

struct SingArgs {
  int n_pairs, n;
  const int *ea, *eb;
  const unsigned char *map_a, *map_b;
  const double *gx, *gw;
  double* out;  // compact blocks [item][la][lb] (scattered by k_sing_scatter)
};

constexpr int kSingLmax = 16; // 8 setup tasks per line: one round of 128 threads
// NTH threads per CTA: 128, or 96 when a chunk holds <= 96 points (n = 6: 16
// lines x 6), so no warp idles through the point phase and 5 CTAs fit an SM
template <class KT, int NTH = 128>
struct SingLayout {
  static constexpr int NL = KT::NL, NC = KT::NC, CH = KT::CHUNK, TS = KT::TS;
  static constexpr int NTR = NL / TS, NT = NTR * NTR, SL = NTH / NT;
  static constexpr int STR = ((NC * NL) % 2 == 0) ? NC * NL + 1 : NC * NL;
  static constexpr int SW = sizeof(typename KT::S) / 8;
  static constexpr int HEAD = 104 * 2 + 2 * KT::TABN + 128;
  static constexpr int STAGE = CH * STR * (SW + 1);
  static constexpr int RED = SL * NL * NL * SW;
  static constexpr int R1 = CH * STR * SW + 2 * kSingLmax * (NL + 1) + 2 * kSingLmax * NL * SW;  // rank-1 path
  static constexpr int BODY0 = STAGE > RED ? STAGE : RED;
  static constexpr int BODY1 = (KT::KIND != 2 && R1 > BODY0) ? R1 : BODY0;
  static constexpr int BODY = (BODY1 + 1) & ~1;  // keeps the setup lines 16 B aligned
  static constexpr int LMAX = kSingLmax;    // rule lines per chunk (setup capacity)
  // real kernels with up to 9 local functions fit 128 registers: 4 CTAs / SM
  static constexpr int kSingMinb = 4;
  static constexpr int kSingMinb16 = 4;
  static constexpr int kSingMinbM = 1;
  static constexpr int kSingMinbH = 4;
  static constexpr int kSingMinb96 = 5;
  static constexpr int MINB = (NTH == 96)                     ? (NL <= 9 && KT::KIND != 2 ? kSingMinb96 : 1)
                              : (KT::KIND == 0 && NL <= 9)    ? kSingMinb
                              : (KT::KIND == 0 && NL <= 16) ? kSingMinb16
                              : (KT::KIND == 1 && NL <= 9)  ? kSingMinbH
                              : (KT::KIND == 2 && NL <= 12) ? kSingMinbM
                                                            : 1;
  // per line: [element][component][A0..4, B0..4] (80), the affine rule
  // descriptor (c0, c1) x 4 + weight (9); odd stride (the lines of one warp
  // read distinct banks)
  static constexpr int LSTRIDE = 2 * 4 * 10 + 10;  // even: 16 B aligned lines (20-bank offset per line)
  static constexpr int SETUP = LMAX * LSTRIDE;
  static constexpr size_t BYTES = static_cast<size_t>(HEAD + BODY + SETUP) * 8;
  static_assert(NL % TS == 0, "tile");
  static_assert(NT <= NTH, "tiles");
};
// the 96-thread variant serves chunks of <= 96 points of Helmholtz kernels with
// up to 9 local functions (measured: Helmholtz q = 2 edge / vertex -3..-4 %;
// real q = 2 +1..2 %, so real kernels keep 128 threads)
template <class KT>
constexpr bool sing96_ok() {
  return KT::KIND == 1 && KT::NL <= 9;
}
inline bool sing96_use(int n) { return (kSingLmax < 128 / n ? kSingLmax : 128 / n) * n <= 96; }

template <class KT, int CLS, int NTH = 128, bool DMMA = false>
__global__ void __launch_bounds__(NTH, SingLayout<KT, NTH>::MINB) k_singular(GeoArgs g, SingArgs A) {
  using S = typename KT::S;
  using LY = SingLayout<KT, NTH>;
  constexpr int NL = KT::NL, NC = KT::NC, CH = LY::CH, TS = LY::TS, NTR = LY::NTR, NT = LY::NT,
                SL = LY::SL, STR = LY::STR;
  extern __shared__ __align__(16) double sm[];
  double* cfa = sm;
  double* cfb = sm + 104;
  double* taba = sm + 208;
  double* tabb = taba + KT::TABN;
  double* gx = tabb + KT::TABN;
  double* gw = gx + 64;
  double* body = gw + 64;
  S* Ga = reinterpret_cast<S*>(body);
  double* Fb = body + CH * STR * LY::SW;
  double* setup = body + LY::BODY;

  const int tid = threadIdx.x;
  const int pr = blockIdx.x;
  const int ea = A.ea[pr], eb = A.eb[pr];
  const int ma = A.map_a[pr], mb = A.map_b[pr];
  const int cella = g.el_cell[ea], cellb = g.el_cell[eb];
  const int n1 = 1 << g.level;
  const int ra = ea % g.epp, rb = eb % g.epp;
  const int ixa = ra % n1, iya = ra / n1, ixb = rb % n1, iyb = rb / n1;
  for (int i = tid; i < 104; i += NTH) {
    cfa[i] = g.cells[static_cast<size_t>(cella) * kCellStride + i];
    cfb[i] = g.cells[static_cast<size_t>(cellb) * kCellStride + i];
  }
  load_tables<KT>(taba, g.tab_a, g.tab_b, ixa, iya, tid, NTH);
  load_tables<KT>(tabb, g.tab_a, g.tab_b, ixb, iyb, tid, NTH);
  const int n = A.n;
  if (tid < n) {
    gx[tid] = A.gx[tid];
    gw[tid] = A.gw[tid];
  }
  __syncthreads();
  const double h = g.h;
  const double sxa = ixa * h - cfa[100], sya = iya * h - cfa[101];
  const double sxb = ixb * h - cfb[100], syb = iyb * h - cfb[101];
  const double h4 = h * h * h * h;
  const int n4 = n * n * n * n;
  // coincident items (same element, equal maps): the integrand is symmetric
  // under exchanging the two points, so half the sectors give C and the block
  // is C + C^T (the Galerkin symmetry the reference tests, test_assembly.cpp:20-29)
  const bool half = CLS == 3 && ma == mb;
  // an element fixed along every rule line: vertex (a), edge with lines over i3
  constexpr bool kFixedEl = CLS == 1 || CLS == 2;
  // scalar shapes with a fixed element: the line's contribution is rank one,
  // s_fixed (x) sum_k gwt_k s_moving,k (or its transpose), so the points stage
  // gwt s_moving only and the block takes one outer product per line
  // (measured: P = 4 edge -12 %, vertex -21 %; Helmholtz q = 2 -1..-3 %; real
  // q = 2 (nl = 9) +2..4 %, where the point-wise GEMM is only ~23 % of the time)
  constexpr bool kRank1 = kFixedEl && KT::KIND != 2 && NC == 1 && (NL >= 16 || KT::KIND == 1);
  const int npts = (CLS == 3 ? (half ? 4 : 8) : (CLS == 2 ? 6 : 4)) * n4;

  S acc[TS][TS];
#pragma unroll
  for (int i = 0; i < TS; ++i)
#pragma unroll
    for (int j = 0; j < TS; ++j) acc[i][j] = zero<S>();
  double dm[2][2][2] = {};  // DMMA path: 2 x 2 tiles of the block, two accumulators each
  if constexpr (DMMA) {     // zero the staging columns a last k-step may read past the chunk
    static_assert(2 * NL * kDmmaPstr <= LY::BODY, "DMMA staging");
    const int pad0 = (min(LY::LMAX, (CH < NTH ? CH : NTH) / A.n) * A.n);
    for (int i = tid; i < ((pad0 + 3) & ~3) - pad0; i += NTH)
      for (int l = 0; l < 2 * NL; ++l) body[l * kDmmaPstr + pad0 + i] = 0.0;
  }
  const int tile = tid % NT, slice = tid / NT;
  const int tr = (tile / NTR) * TS, tc = (tile % NTR) * TS;
  const bool active = slice < SL;

  // chunks of whole rule lines.  Setup: per (line, element, homogeneous
  // component) the inner Horner sums of the jet at the line's fixed coordinate
  // (task (e, c) = (0, 0) also stores the line's affine rule descriptor);
  // then one thread per point finishes both jets from the setup.
  const int nlines = npts / n;
  const int lpc = min(LY::LMAX, (CH < NTH ? CH : NTH) / n), cpts = lpc * n;
  const float rn = 1.0f / static_cast<float>(n);
  const int my_ll = div_n(tid, n, rn), my_k = tid - my_ll * n;  // this thread's point of a chunk
  // phases per chunk: point evaluation | GEMM of this chunk + setup of the next
  // (disjoint shared regions), two barriers per chunk
  auto do_setup = [&](int lb) {
    for (int task = tid; task < lpc * 8; task += NTH) {
      // classes with a fixed element (vertex; edge over i3): element-major task
      // order (e warp-uniform when 4 lpc is a multiple of 32: the two elements'
      // tasks differ); else line-major (fewer bank conflicts on the setup stores)
      int e, ll, c;
      if (kFixedEl) {
        e = task >= lpc * 4;
        const int rem = task - e * lpc * 4;
        ll = rem >> 2;
        c = rem & 3;
      } else {
        ll = task >> 3;
        e = (task >> 2) & 1;
        c = task & 3;
      }
      const int line = lb + ll;
      if (line < nlines) {
        double c0[4], c1[4], wl;
        rule_line<CLS>(line, n, rn, gx, gw, ma, mb, c0, c1, wl, half);
        // the moving parameter of element e is the one with c1 != 0
        const int vm = e ? (c1[3] != 0.0) : (c1[1] != 0.0);
        const double sx0 = e ? sxb : sxa, sy0 = e ? syb : sya;
        const double f = vm ? sx0 + h * c0[2 * e] : sy0 + h * c0[2 * e + 1];
        double* L = setup + ll * LY::LSTRIDE;
        if (kFixedEl && (CLS == 1 ? e == 0 : (c1[2 * e] == 0.0 && c1[2 * e + 1] == 0.0))) {  // e fixed on the line
          double res[10], N, Ns, Nt;
          jet_setup_regs((e ? cfb : cfa) + c * 25, vm, f, res);
          jet_comp(res, vm, vm ? sy0 + h * c0[2 * e + 1] : sx0 + h * c0[2 * e], N, Ns, Nt);
          double* Le = L + (e * 4 + c) * 10;
          Le[0] = N;
          Le[1] = Ns;
          Le[2] = Nt;
        } else {
          jet_setup((e ? cfb : cfa) + c * 25, vm, f, L + (e * 4 + c) * 10);
        }
        if (e == 0 && c == 0) {
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            reinterpret_cast<double2*>(L + 80)[k] = make_double2(c0[k], c1[k]);
          }
          L[88] = wl;
        }
      }
    }
  };
  do_setup(0);
  __syncthreads();
  // rank-1 path: s_fixed + orientation [2][LMAX][NL + 1] and line sums
  // [2][LMAX][NL] double-buffered by chunk, so chunk c's outer products run in
  // the point phase of chunk c + 1 (two barriers per chunk)
  double* Fr = Fb;
  S* Vr = reinterpret_cast<S*>(Fr + 2 * LY::LMAX * (NL + 1));
  auto gemm1 = [&](int bsel) {
    if (!active) return;
    for (int ll = slice; ll < lpc; ll += SL) {
      const double* f = Fr + (bsel * LY::LMAX + ll) * (NL + 1);
      const S* v = Vr + (bsel * LY::LMAX + ll) * NL;
      if (f[NL] != 0.0) {  // a fixed: rows s_fixed, columns the line sum
        double fr[TS];
        S vc[TS];
#pragma unroll
        for (int i = 0; i < TS; ++i) {
          fr[i] = f[tr + i];
          vc[i] = v[tc + i];
        }
#pragma unroll
        for (int i = 0; i < TS; ++i)
#pragma unroll
          for (int j = 0; j < TS; ++j) fmac(acc[i][j], vc[j], fr[i]);
      } else {  // b fixed: rows the line sum, columns s_fixed
        S vr[TS];
        double fc[TS];
#pragma unroll
        for (int i = 0; i < TS; ++i) {
          vr[i] = v[tr + i];
          fc[i] = f[tc + i];
        }
#pragma unroll
        for (int i = 0; i < TS; ++i)
#pragma unroll
          for (int j = 0; j < TS; ++j) fmac(acc[i][j], vr[i], fc[j]);
      }
    }
  };
  (void)gemm1;
  int rb1 = 0;
  for (int lbase = 0; lbase < nlines; lbase += lpc, rb1 ^= 1) {
    if (tid < cpts) {
      const int p = lbase * n + tid;
      S* ga = Ga + tid * STR;
      double* fb = Fb + tid * STR;
      if (p < npts) {
        const double* L = setup + my_ll * LY::LSTRIDE;
        const double gk4 = gx[my_k];
        const double2* D = reinterpret_cast<const double2*>(L + 80);
        const double2 du_ = D[0], dv_ = D[1], dub_ = D[2], dvb_ = D[3];
        const double ua = fma(du_.y, gk4, du_.x), va = fma(dv_.y, gk4, dv_.x);
        const double ub = fma(dub_.y, gk4, dub_.x), vb = fma(dvb_.y, gk4, dvb_.x);
        const int vma = dv_.y != 0.0, vmb = dvb_.y != 0.0;
        const double w = L[88] * gw[my_k];
        const double sa_ = sxa + h * ua, ta_ = sya + h * va, sb_ = sxb + h * ub, tb_ = syb + h * vb;
        double xa[3], dua[3], dva[3], xb[3], dub[3], dvb[3];
        // vertex: a always fixed, b never; edge: per line (kind 1 fixes b)
        const bool fa = kFixedEl && (CLS == 1 || (du_.y == 0.0 && dv_.y == 0.0));
        const bool fbx = kFixedEl && CLS != 1 && dub_.y == 0.0 && dvb_.y == 0.0;
        if constexpr (kFixedEl) {
          if (fa)
            jet_fixed(L, xa, dua, dva);
          else
            jet_line(L, vma, vma ? ta_ : sa_, xa, dua, dva);
          if (fbx)
            jet_fixed(L + 40, xb, dub, dvb);
          else
            jet_line(L + 40, vmb, vmb ? tb_ : sb_, xb, dub, dvb);
        } else {
          jet_line(L, vma, vma ? ta_ : sa_, xa, dua, dva);
          jet_line(L + 40, vmb, vmb ? tb_ : sb_, xb, dub, dvb);
        }
        const double sga = sqrt_g_of(dua, dva), sgb = sqrt_g_of(dub, dvb);
        const double d0 = xa[0] - xb[0], d1 = xa[1] - xb[1], d2 = xa[2] - xb[2];
        const S gk = green_k<KT>(d0 * d0 + d1 * d1 + d2 * d2, g.kp);
        const double wt = w * sga * sgb * h4;
        const S gwt = gk * wt;
        double sa[NC][NL], sb[NC][NL];
        shapes<KT>(taba, ua, va, h, dua, dva, sga, sa);
        shapes<KT>(tabb, ub, vb, h, dub, dvb, sgb, sb);
        if constexpr (kRank1) {
          // ga holds gwt s_moving; the line's first point stores s_fixed + orientation
#pragma unroll
          for (int l = 0; l < NL; ++l) ga[l] = gwt * (fa ? sb[0][l] : sa[0][l]);
          if (my_k == 0) {
            double* f = Fr + (rb1 * LY::LMAX + my_ll) * (NL + 1);
#pragma unroll
            for (int l = 0; l < NL; ++l) f[l] = fa ? sa[0][l] : sb[0][l];
            f[NL] = fa ? 1.0 : 0.0;
          }
        } else {
          (void)fbx;
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            S wc = gwt;
            if constexpr (KT::KIND == 2) {
              if (c == 3) wc = gwt * mk(g.kp.dwx, g.kp.dwy);
            }
#pragma unroll
            for (int l = 0; l < NL; ++l) {
              if constexpr (DMMA) {  // transposed staging [l][point]: conflict-free DMMA fragments
                reinterpret_cast<double*>(body)[l * kDmmaPstr + tid] = wc * sa[c][l];
                body[(NL + l) * kDmmaPstr + tid] = sb[c][l];
              } else {
                ga[c * NL + l] = wc * sa[c][l];
                fb[c * NL + l] = sb[c][l];
              }
            }
          }
        }
      } else {
        if constexpr (kRank1) {
#pragma unroll
          for (int l = 0; l < NL; ++l) ga[l] = zero<S>();
          if (my_k == 0) {
            double* f = Fr + (rb1 * LY::LMAX + my_ll) * (NL + 1);
#pragma unroll
            for (int l = 0; l <= NL; ++l) f[l] = 0.0;
          }
        } else {
#pragma unroll
          for (int c = 0; c < NC * NL; ++c) {
            if constexpr (DMMA) {
              body[c * kDmmaPstr + tid] = 0.0;
              body[(NL + c) * kDmmaPstr + tid] = 0.0;
            } else {
              ga[c] = zero<S>();
              fb[c] = 0.0;
            }
          }
        }
      }
    }
    if constexpr (kRank1) {
      if (lbase > 0) gemm1(rb1 ^ 1);
    }
    __syncthreads();
    if constexpr (kRank1) {
      // line sums V[ll][l] = sum_k gwt_k s_moving,k[l] (fixed order)
      for (int task = tid; task < lpc * NL; task += NTH) {
        const int ll = task / NL, l = task - ll * NL;
        const S* m = Ga + ll * n * STR + l;
        S sum = zero<S>();
        for (int k = 0; k < n; ++k) sum = sum + m[k * STR];
        Vr[(rb1 * LY::LMAX + ll) * NL + l] = sum;
      }
    } else if constexpr (DMMA) {
      // Ga^T (NL x points) . Fb (points x NL) on the FP64 tensor cores: the
      // warps take k-steps of 4 points round-robin, 2 x 2 tiles of 8 x 8
      static_assert(KT::KIND == 0 && NC == 1 && NL == 16, "DMMA accumulation: real, 16 local functions");
      const int wv = tid >> 5, ln = tid & 31, gid = ln >> 2, tig = ln & 3;
      for (int st = wv; st * 4 < cpts; st += NTH / 32) {
        const double* gr = body + gid * kDmmaPstr + st * 4 + tig;
        const double* fr = body + (NL + gid) * kDmmaPstr + st * 4 + tig;
        const double a0 = gr[0], a1 = gr[8 * kDmmaPstr], b0 = fr[0], b1 = fr[8 * kDmmaPstr];
        dmma884(dm[0][0], a0, b0);
        dmma884(dm[0][1], a0, b1);
        dmma884(dm[1][0], a1, b0);
        dmma884(dm[1][1], a1, b1);
      }
    } else if (active) {
      for (int pt = slice; pt < cpts; pt += SL) {
        const S* ga = Ga + pt * STR;
        const double* fb = Fb + pt * STR;
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          S av[TS];
          double bv[TS];
#pragma unroll
          for (int i = 0; i < TS; ++i) {
            av[i] = ga[c * NL + tr + i];
            bv[i] = fb[c * NL + tc + i];
          }
#pragma unroll
          for (int i = 0; i < TS; ++i)
#pragma unroll
            for (int j = 0; j < TS; ++j) fmac(acc[i][j], av[i], bv[j]);
        }
      }
    }
    if (lbase + lpc < nlines) do_setup(lbase + lpc);
    __syncthreads();
  }
  if constexpr (kRank1) {
    gemm1(rb1 ^ 1);
    __syncthreads();
  }
  S* red = reinterpret_cast<S*>(body);
  constexpr int NSL = DMMA ? NTH / 32 : SL;  // partial blocks: warps (DMMA) or slices
  if constexpr (DMMA) {
    const int wv = tid >> 5, ln = tid & 31, gid = ln >> 2, tig = ln & 3;
    double* rd = reinterpret_cast<double*>(red) + wv * NL * NL;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        rd[(8 * i + gid) * NL + 8 * j + 2 * tig] = dm[i][j][0];
        rd[(8 * i + gid) * NL + 8 * j + 2 * tig + 1] = dm[i][j][1];
      }
  } else if (active) {
#pragma unroll
    for (int i = 0; i < TS; ++i)
#pragma unroll
      for (int j = 0; j < TS; ++j) red[(slice * NL + tr + i) * NL + tc + j] = acc[i][j];
  }
  __syncthreads();
  S* out = reinterpret_cast<S*>(A.out) + static_cast<size_t>(pr) * NL * NL;
  for (int o = tid; o < NL * NL; o += NTH) {
    S v = zero<S>();
    for (int s = 0; s < NSL; ++s) v = v + red[s * NL * NL + o];
    if (half) {
      const int ot = (o % NL) * NL + o / NL;
#pragma unroll 1
      for (int s = 0; s < NSL; ++s) v = v + red[s * NL * NL + ot];
    }
    out[o] = v;
  }
}

}  // namespace dev
// one launch of a singular class: 96-thread CTAs when the chunk holds <= 96 points
template <class KT, int CLS>
void launch_singular(const dev::GeoArgs& g, const dev::SingArgs& A, cudaStream_t st) {
  if constexpr (dev::sing96_ok<KT>()) {
    if (dev::sing96_use(A.n)) {
      using LY = dev::SingLayout<KT, 96>;
      IGB_CUDA(cudaFuncSetAttribute(dev::k_singular<KT, CLS, 96>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    static_cast<int>(LY::BYTES)));
      dev::k_singular<KT, CLS, 96><<<A.n_pairs, 96, LY::BYTES, st>>>(g, A);
      return;
    }
  }
  using LY = dev::SingLayout<KT, 128>;
  if constexpr (KT::KIND == 0 && KT::NL == 16 && CLS == 3) {
    // real, 16 local functions, point-wise accumulation: on the FP64 tensor
    // cores (c5 coincident 286 -> 245 ms; ncu: profiles/r02_ncu_c5_sing_summary.md)
    IGB_CUDA(cudaFuncSetAttribute(dev::k_singular<KT, CLS, 128, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(LY::BYTES)));
    dev::k_singular<KT, CLS, 128, true><<<A.n_pairs, 128, LY::BYTES, st>>>(g, A);
  } else {
    IGB_CUDA(cudaFuncSetAttribute(dev::k_singular<KT, CLS, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  static_cast<int>(LY::BYTES)));
    dev::k_singular<KT, CLS, 128><<<A.n_pairs, 128, LY::BYTES, st>>>(g, A);
  }
}
namespace dev {
// Singular blocks are integrated before the block partition exists (they only
// need the mesh topology); once the near list is known each item's block goes
// to the slot of (ea, eb) and its transpose to the slot of (eb, ea) (the
// bilinear forms are symmetric: spaces.cpp singular pairs are computed once).
template <class S, int NL>
__global__ void __launch_bounds__(128) k_sing_scatter(const int* __restrict__ slot_ab, const int* __restrict__ slot_ba,
                                                      const int* __restrict__ near_a, const int* __restrict__ near_rs,
                                                      const S* __restrict__ blk, S* __restrict__ near) {
  __shared__ S tr[NL][NL + 1];
  const int k = blockIdx.x;
  const S* b = blk + static_cast<size_t>(k) * NL * NL;
  const int qab = slot_ab[k], qba = slot_ba[k];
  for (int o = threadIdx.x; o < NL * NL; o += blockDim.x) {
    const int la = o / NL, lb = o % NL;
    const S v = b[o];
    tr[la][lb] = v;
    if (qab >= 0) near[near_off(near_a, near_rs, qab, la, lb, NL)] = v;
  }
  if (qba < 0 || qba == qab) return;  // block-uniform
  __syncthreads();
  for (int o = threadIdx.x; o < NL * NL; o += blockDim.x) {
    const int r = o / NL, c = o % NL;
    near[near_off(near_a, near_rs, qba, r, c, NL)] = tr[c][r];
  }
}

// --------------------------------------------------------- K6: matvec
template <class S>
__global__ void k_coef(int n, const S* __restrict__ x, const int* __restrict__ l2g, const double* __restrict__ sg,
                       S* __restrict__ coef) {
  pdl_entry();  // h2.cpp:271-279
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) coef[i] = x[l2g[i]] * sg[i];
}
__device__ __forceinline__ double operator_mul(double a, double b) { return a * b; }

template <class S, int NL>
__global__ void k_leaf_up(int n_el, const int* __restrict__ el, int rows, int epp, int npp, int leaf_off,
                          const double* __restrict__ mom, const S* __restrict__ coef,
                          S* __restrict__ up) {
  pdl_entry();  // h2.cpp:281-290, owned leaves
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_el) * rows) return;
  const int e = el[idx / rows], r = static_cast<int>(idx % rows);
  S acc = zero<S>();
#pragma unroll
  for (int l = 0; l < NL; ++l)
    fmac(acc, coef[static_cast<size_t>(e) * NL + l], __ldg(mom + (static_cast<size_t>(e) * NL + l) * rows + r));
  const int leaf = (e / epp) * npp + leaf_off + (e % epp);
  up[static_cast<size_t>(leaf) * rows + r] = acc;
}

// leaf moments straight from x (coefficients gathered inline: h2.cpp:271-290)
// and, in the same launch, down := 0 (level-split graph)
template <class S, int NL>
__global__ void k_leaf_up_x(int n_el, int rows, int epp, int npp, int leaf_off, const double* __restrict__ mom,
                            const S* __restrict__ x, const int* __restrict__ l2g, const double* __restrict__ sg,
                            S* __restrict__ up, S* __restrict__ down, long long ndown) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx < ndown) down[idx] = zero<S>();
  if (idx >= static_cast<long long>(n_el) * rows) return;
  const int e = static_cast<int>(idx / rows), r = static_cast<int>(idx % rows);
  S acc = zero<S>();
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int k = e * NL + l;
    fmac(acc, x[l2g[k]] * sg[k], __ldg(mom + static_cast<size_t>(k) * rows + r));
  }
  const int leaf = (e / epp) * npp + leaf_off + (e % epp);
  up[static_cast<size_t>(leaf) * rows + r] = acc;
}

// node of a level-l tree in level-1 cluster c (l >= 1), local index sc
__device__ __forceinline__ void cluster_node(int c, int level, int sc, int& p, int& sx, int& sy) {
  const int half = 1 << (level - 1);
  const int k1 = c & 3;
  p = c >> 2;
  sx = (k1 & 1) * half + sc % half;
  sy = (k1 >> 1) * half + sc / half;
}

// parent(i,j) = sum_k tu_k X_k tv_k^T  (h2.cpp:291-310); level 0: all roots,
// level >= 1: the nodes of level-1 clusters [c0, c1).  M > 0: compile-time
// interpolation degree (loops unrolled, all child loads in flight at once);
// M = 0: runtime m.
template <class S, int M>
__global__ void k_up_level(int np, int level, int npp, int off_l, int off_c, int m_rt, int nch,
                           const double* __restrict__ tl, const double* __restrict__ tr, S* __restrict__ up, int c0,
                           int c1) {
  pdl_entry();
  const int m = M ? M : m_rt;
  const int mm = m * m, rows = nch * mm, nside = 1 << level;
  const int per = level == 0 ? 1 : (1 << (2 * (level - 1)));
  const int ncl = level == 0 ? np : (c1 - c0);
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(ncl) * per * rows) return;
  const int r = static_cast<int>(idx % rows);
  const long long nidx = idx / rows;
  const int ci = static_cast<int>(nidx / per), sc = static_cast<int>(nidx % per);
  int p, sx, sy;
  if (level == 0) {
    p = ci;
    sx = sy = 0;
  } else {
    cluster_node(c0 + ci, level, sc, p, sx, sy);
  }
  const int c = r / mm, nu = r % mm, i = nu % m, j = nu / m;
  const int cside = nside * 2;
  S acc = zero<S>();
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int child = p * npp + off_c + (2 * sx + (k & 1)) + cside * (2 * sy + (k >> 1));
    const double* tu = (k & 1) ? tr : tl;
    const double* tv = (k >> 1) ? tr : tl;
    const S* X = up + static_cast<size_t>(child) * rows + c * mm;
#pragma unroll
    for (int b = 0; b < m; ++b) {
      S t = zero<S>();
#pragma unroll
      for (int a = 0; a < m; ++a) fmac(t, X[a + m * b], __ldg(tu + i + m * a));
      fmac(acc, t, __ldg(tv + j + m * b));
    }
  }
  up[static_cast<size_t>(p * npp + off_l + sx + nside * sy) * rows + r] = acc;
}

// down[t] = sum_q w_c K_q up[tb_q]  (h2.cpp:312-326); one warp per target
template <class S, int NCH, int R>
__global__ void __launch_bounds__(256) k_far(int n_targets, const int* __restrict__ targets,
                                             const int* __restrict__ far_rs, const int* __restrict__ far_b,
                                             const S* __restrict__ K, int mm, const S* __restrict__ up,
                                             S dw, S* __restrict__ down) {
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_targets) return;
  const int t = targets[warp];
  const int rows = NCH * mm;
  const int G = (mm <= 32) ? 32 / mm : 1;
  const int g = (mm <= 32) ? lane / mm : 0;
  const int nu0 = (mm <= 32) ? lane % mm : lane;
  const bool ok = g < G;
  S acc[NCH][R];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[c][r] = zero<S>();
  const int q0 = far_rs[t], q1 = far_rs[t + 1];
  if (ok) {
    for (int q = q0 + g; q < q1; q += G) {
      const S* Kq = K + static_cast<size_t>(q) * mm * mm;
      const S* src = up + static_cast<size_t>(far_b[q]) * rows;
      S part[NCH][R];
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int r = 0; r < R; ++r) part[c][r] = zero<S>();
#pragma unroll 4
      for (int mu = 0; mu < mm; ++mu) {
        S xv[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) xv[c] = src[c * mm + mu];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int nu = nu0 + 32 * r;
          if (nu < mm) {
            const S kv = ldg_s(Kq + mu * mm + nu);
#pragma unroll
            for (int c = 0; c < NCH; ++c) fmac(part[c][r], kv, xv[c]);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if (NCH == 4 && c == 3)
            acc[c][r] = acc[c][r] + part[c][r] * dw;
          else
            acc[c][r] = acc[c][r] + part[c][r];
        }
    }
  }
  // combine the G lane groups in fixed order
  for (int gg = 1; gg < G; ++gg) {
    const int src = (lane + gg * mm < 32) ? lane + gg * mm : lane;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const S v = shfl_idx(acc[c][0], src);
      if (g == 0) acc[c][0] = acc[c][0] + v;
    }
  }
  if (g == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int nu = nu0 + 32 * r;
      if (nu < mm)
#pragma unroll
        for (int c = 0; c < NCH; ++c) down[static_cast<size_t>(t) * rows + c * mm + nu] = acc[c][r];
    }
  }
}

// Stored-coupling far field, one CTA per target (h2.cpp:312-326): its 8 warps
// take the target's pairs round-robin (each streams a pair's m^2 x m^2 block
// with lanes on rows nu, 8 coupling loads in flight per lane), and the warps'
// partial sums are added in fixed warp order through shared memory.  Balances
// targets with ~190 pairs against those with a few (the warp-per-target
// kernel left c4 at 49 % of HBM).
template <class S, int NCH, int R>
__global__ void __launch_bounds__(256, 2) k_far_cta(const int* __restrict__ targets, const int* __restrict__ far_rs,
                                                 const int* __restrict__ far_b, const S* __restrict__ K, int mm,
                                                 const S* __restrict__ up, S dw, S* __restrict__ down) {
  extern __shared__ __align__(16) double far_cta_sh[];
  S* part_sh = reinterpret_cast<S*>(far_cta_sh);  // [warp][c * mm + nu]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int t = targets[blockIdx.x];
  const int rows = NCH * mm;
  S acc[NCH][R];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[c][r] = zero<S>();
  const int q1 = far_rs[t + 1];
  constexpr int B = 16 / R;  // coupling columns loaded per batch: 16 loads in flight per lane
  for (int q = far_rs[t] + w; q < q1; q += 8) {
    const S* Kq = K + static_cast<size_t>(q) * mm * mm;
    const S* src = up + static_cast<size_t>(__ldg(far_b + q)) * rows;
    for (int mu0 = 0; mu0 < mm; mu0 += B) {
      S kv[B][R];
#pragma unroll
      for (int j = 0; j < B; ++j)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const int nu = lane + 32 * r, mu = mu0 + j;
          kv[j][r] = (nu < mm && mu < mm) ? ldg_s(Kq + static_cast<size_t>(mu) * mm + nu) : zero<S>();
        }
#pragma unroll
      for (int j = 0; j < B; ++j) {
        if (mu0 + j >= mm) break;
        S xv[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) xv[c] = ldg_s(src + c * mm + mu0 + j);
#pragma unroll
        for (int r = 0; r < R; ++r)
#pragma unroll
          for (int c = 0; c < NCH; ++c) fmac(acc[c][r], kv[j][r], xv[c]);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = lane + 32 * r;
    if (nu < mm)
#pragma unroll
      for (int c = 0; c < NCH; ++c) part_sh[static_cast<size_t>(w) * rows + c * mm + nu] = acc[c][r];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < rows; i += blockDim.x) {
    S v = part_sh[i];
#pragma unroll
    for (int ww = 1; ww < 8; ++ww) v = v + part_sh[static_cast<size_t>(ww) * rows + i];
    if (NCH == 4 && i >= 3 * mm) v = v * dw;  // divergence channel weight -kappa^-2
    down[static_cast<size_t>(t) * rows + i] = v;
  }
}

// Fused far field: couplings evaluated on the fly from the L2-resident node
// images, K_q[nu][mu] = G(|img_t[nu] - img_s[mu]|) (h2.cpp:218-229), applied
// as in h2.cpp:312-326.  One warp per target; G lane groups take alternate
// source clusters; each source's images + moments are staged once per warp in
// shared memory and read back as broadcasts.  No coupling bytes touch HBM.
template <class KT, int R>
__global__ void __launch_bounds__(256) k_far_fused(int n_targets, const int* __restrict__ targets,
                                                   const int* __restrict__ far_rs, const int* __restrict__ far_b,
                                                   const double* __restrict__ img, int mm,
                                                   const typename KT::S* __restrict__ up, KParams kp,
                                                   typename KT::S* __restrict__ down) {
  using S = typename KT::S;
  constexpr int NCH = KT::NC;
  constexpr int SW = sizeof(S) / 8;
  constexpr int PW = ((4 + NCH * SW) + 1) / 2 * 2;  // x, y, z, pad, moments; even => 16 B aligned
  extern __shared__ __align__(16) double smf[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double* wsm = smf + static_cast<size_t>(wib) * 32 * R * PW;
  if (warp >= n_targets) return;
  const int t = targets[warp];
  const int rows = NCH * mm;
  const int G = (mm <= 32) ? 32 / mm : 1;
  const int g = (mm <= 32) ? lane / mm : 0;
  const int lig = (mm <= 32) ? lane % mm : lane;  // lane index within the group
  const bool ok = g < G;
  double* gsm = wsm + static_cast<size_t>(g < G ? g : 0) * mm * PW;
  double tx[R][3];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = lig + 32 * r;
    const double* p = img + (static_cast<size_t>(t) * mm + (nu < mm ? nu : 0)) * 3;
    tx[r][0] = p[0];
    tx[r][1] = p[1];
    tx[r][2] = p[2];
  }
  S acc[NCH][R];
#pragma unroll
  for (int c = 0; c < NCH; ++c)
#pragma unroll
    for (int r = 0; r < R; ++r) acc[c][r] = zero<S>();
  const int q0 = far_rs[t], q1 = far_rs[t + 1];
  for (int base = q0; base < q1; base += G) {
    const int q = base + g;
    const bool valid = ok && q < q1;
    if (valid) {
      const int s = far_b[q];
      const double* is = img + static_cast<size_t>(s) * mm * 3;
      const S* us = up + static_cast<size_t>(s) * rows;
      for (int mu = lig; mu < mm; mu += (mm <= 32 ? mm : 32)) {
        double* d = gsm + mu * PW;
        d[0] = is[3 * mu];
        d[1] = is[3 * mu + 1];
        d[2] = is[3 * mu + 2];
#pragma unroll
        for (int c = 0; c < NCH; ++c) reinterpret_cast<S*>(d + 4)[c] = us[c * mm + mu];
      }
    }
    __syncwarp();
    if (valid) {
      S part[NCH][R];
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int r = 0; r < R; ++r) part[c][r] = zero<S>();
#pragma unroll 2
      for (int mu = 0; mu < mm; ++mu) {
        const double* d = gsm + mu * PW;
        const double2 xy = *reinterpret_cast<const double2*>(d);
        const double sz = d[2];
        S xv[NCH];
#pragma unroll
        for (int c = 0; c < NCH; ++c) xv[c] = reinterpret_cast<const S*>(d + 4)[c];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const double d0 = tx[r][0] - xy.x, d1 = tx[r][1] - xy.y, d2 = tx[r][2] - sz;
          const S gk = green_far<KT>(d0 * d0 + d1 * d1 + d2 * d2, kp);
#pragma unroll
          for (int c = 0; c < NCH; ++c) fmac(part[c][r], gk, xv[c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c)
#pragma unroll
        for (int r = 0; r < R; ++r) {
          if constexpr (NCH == 4) {
            if (c == 3) {
              acc[c][r] = acc[c][r] + part[c][r] * mk(kp.dwx, kp.dwy);
              continue;
            }
          }
          acc[c][r] = acc[c][r] + part[c][r];
        }
    }
    __syncwarp();
  }
  for (int gg = 1; gg < G; ++gg) {
    const int src = (lane + gg * mm < 32) ? lane + gg * mm : lane;
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const S v = shfl_idx(acc[c][0], src);
      if (g == 0) acc[c][0] = acc[c][0] + v;
    }
  }
  if (g == 0) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int nu = lig + 32 * r;
      if (nu < mm)
#pragma unroll
        for (int c = 0; c < NCH; ++c) down[static_cast<size_t>(t) * rows + c * mm + nu] = acc[c][r];
    }
  }
}

// Symmetric fused far field, warp-row layout (complex kinds, Maxwell channels,
// m >= 6): K(s,t) = K(t,s)^T, so each unordered admissible pair {t, s}, t < s,
// is evaluated once by the warp of t.  Lane owns target rows nu = lane + 32 r;
// the source cluster's points and moments are staged in shared memory; per
// source point mu each lane accumulates K up[s] into its rows and its share of
// (K^T up[t])[mu], which a fixed xor tree sums over the warp.  The products
// (channel weight w_c applied, Maxwell: -1/kappa^2 on the divergence channel)
// go to the slot of the transposed pair, summed by k_far_lower.
template <class KT, int R>
__global__ void __launch_bounds__(256) k_far_sym_w(int n_targets, const int* __restrict__ targets,
                                                   const int* __restrict__ upper_start,
                                                   const int* __restrict__ far_rs, const int* __restrict__ far_b,
                                                   const int* __restrict__ trans, const double* __restrict__ img,
                                                   int mm, const typename KT::S* __restrict__ up, KParams kp,
                                                   typename KT::S* __restrict__ down,
                                                   typename KT::S* __restrict__ slot) {
  using S = typename KT::S;
  constexpr int NCH = KT::NC;
  constexpr int SW = sizeof(S) / 8;
  constexpr int PW = ((4 + NCH * SW) + 1) / 2 * 2;
  extern __shared__ __align__(16) double smf[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  double* gsm = smf + static_cast<size_t>(wib) * 32 * R * PW;
  if (warp >= n_targets) return;
  const int t = targets[warp];
  const int rows = NCH * mm;
  S wc[NCH];
#pragma unroll
  for (int c = 0; c < NCH; ++c) wc[c] = (NCH == 4 && c == 3) ? mk_s<S>(kp.dwx, kp.dwy) : mk_s<S>(1.0, 0.0);
  double tx[R][3];
  S xt[R][NCH], acc[NCH][R];
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = lane + 32 * r;
    const bool ok = nu < mm;
    const double* p = img + (static_cast<size_t>(t) * mm + (ok ? nu : 0)) * 3;
    tx[r][0] = p[0];
    tx[r][1] = p[1];
    tx[r][2] = p[2];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      xt[r][c] = ok ? up[static_cast<size_t>(t) * rows + c * mm + nu] : zero<S>();
      acc[c][r] = zero<S>();
    }
  }
  for (int q = upper_start[t]; q < far_rs[t + 1]; ++q) {
    const int s = far_b[q];
    const double* is = img + static_cast<size_t>(s) * mm * 3;
    const S* us = up + static_cast<size_t>(s) * rows;
    for (int mu = lane; mu < mm; mu += 32) {
      double* d = gsm + mu * PW;
      d[0] = is[3 * mu];
      d[1] = is[3 * mu + 1];
      d[2] = is[3 * mu + 2];
#pragma unroll
      for (int c = 0; c < NCH; ++c) reinterpret_cast<S*>(d + 4)[c] = us[c * mm + mu];
    }
    __syncwarp();
    S pst[NCH][R];
#pragma unroll
    for (int c = 0; c < NCH; ++c)
#pragma unroll
      for (int r = 0; r < R; ++r) pst[c][r] = zero<S>();
    for (int mu = 0; mu < mm; ++mu) {
      const double* d = gsm + mu * PW;
      const double2 xy = *reinterpret_cast<const double2*>(d);
      const double sz = d[2];
      S xs[NCH], v[NCH];
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        xs[c] = reinterpret_cast<const S*>(d + 4)[c];
        v[c] = zero<S>();
      }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (lane + 32 * r >= mm) continue;
        const double d0 = tx[r][0] - xy.x, d1 = tx[r][1] - xy.y, d2 = tx[r][2] - sz;
        const S gk = green_far<KT>(d0 * d0 + d1 * d1 + d2 * d2, kp);
#pragma unroll
        for (int c = 0; c < NCH; ++c) {
          fmac(acc[c][r], gk, xs[c]);
          fmac(v[c], gk, xt[r][c]);
        }
      }
#pragma unroll
      for (int c = 0; c < NCH; ++c) {
        S w = v[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) w = w + shfl_xor(w, o);
        if ((mu & 31) == lane) pst[c][mu >> 5] = w;
      }
    }
    S* dst = slot + static_cast<size_t>(trans[q]) * rows;
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const int mu = lane + 32 * r;
      if (mu < mm)
#pragma unroll
        for (int c = 0; c < NCH; ++c) dst[c * mm + mu] = pst[c][r] * wc[c];
    }
    __syncwarp();
  }
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const int nu = lane + 32 * r;
    if (nu < mm)
#pragma unroll
      for (int c = 0; c < NCH; ++c) down[static_cast<size_t>(t) * rows + c * mm + nu] = acc[c][r] * wc[c];
  }
}


template <int M>
struct SymTile {  // lane grid BR x BC over the (nu, mu) block of one far pair (m = 6)
  static constexpr int MM = M * M;
  static constexpr int BR = 4, BC = 8;
  static constexpr int RN = (MM + BR - 1) / BR, CN = (MM + BC - 1) / BC;
  static_assert(BR * BC <= 32, "lane grid");
};

// 2/r from the MUFU estimate y0 and one Newton step y0 (3 - x y0^2) (the
// factor 1/2 of the step folded into the final scale): relative error
// 1.5 e0^2 for the estimate's e0
__device__ __forceinline__ double far_rsqrt(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  return y0 * fma(-x * y0, y0, 3.0);
}
constexpr double kFarScale = 0.5 * kInv4Pi;

// Symmetric fused far field (Laplace): each unordered admissible pair {t, s},
// t < s, is evaluated once by the warp of t: K = G(|img_t[nu] - img_s[mu]|)
// gives down[t] += K up[s] (accumulated in registers) and K^T up[t], written to
// the slot of the transposed pair (s, t) and summed by k_far_lower in fixed
// order.  Lane (bi, bj) owns RN target rows x CN source columns.
template <int M, bool DIST>
__device__ __forceinline__ void far_sym_body(int n_targets, const int* __restrict__ targets,
                                             const int* __restrict__ upper_start, const int* __restrict__ far_rs,
                                             const int* __restrict__ far_b, const int* __restrict__ trans,
                                             const double* __restrict__ img, const double* __restrict__ up,
                                             double* __restrict__ down, double* __restrict__ slot,
                                             const unsigned char* __restrict__ owned, int full_row) {
  using T = SymTile<M>;
  constexpr int MM = T::MM, BR = T::BR, BC = T::BC, RN = T::RN, CN = T::CN;
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= n_targets) return;
  const int t = targets[warp];
  const int bi = lane % BR, bj = lane / BR;
  const bool act = bj < BC;
  double tx[RN][3], xt[RN], acc[RN];
#pragma unroll
  for (int i = 0; i < RN; ++i) {
    const int nu = bi + BR * i;
    const bool ok = act && nu < MM;
    const double* p = img + (static_cast<size_t>(t) * MM + (ok ? nu : 0)) * 3;
    tx[i][0] = p[0];
    tx[i][1] = p[1];
    tx[i][2] = p[2];
    xt[i] = ok ? up[static_cast<size_t>(t) * MM + nu] : 0.0;
    acc[i] = 0.0;
  }
  // pairs (t, s): s > t and s owned -> symmetric (t's row + slot of (s, t));
  // s not owned (other rank's block rows) -> one-sided; s < t owned -> skip
  // (evaluated by s's warp).  Single GPU: every s owned, only s > t visited.
  const int q0 = (DIST && full_row) ? far_rs[t] : upper_start[t], q1 = far_rs[t + 1];
  double nsx[CN][3], nxs[CN];
  // single GPU: source indices read one pair ahead, so the image loads of pair
  // q depend on a register, not on a load issued in the same iteration
  constexpr bool kAhead = !DIST;
  int s_nx = (kAhead && q0 < q1) ? __ldg(far_b + q0) : 0;
  auto load = [&](int q) {
    int s;
    if constexpr (kAhead) {
      s = s_nx;
      if (q + 1 < q1) s_nx = __ldg(far_b + q + 1);
    } else {
      s = far_b[q];
    }
#pragma unroll
    for (int j = 0; j < CN; ++j) {
      const int mu = bj + BC * j;
      const bool ok = act && mu < MM;
      const double* p = img + (static_cast<size_t>(s) * MM + (ok ? mu : 0)) * 3;
      nsx[j][0] = __ldg(p);
      nsx[j][1] = __ldg(p + 1);
      nsx[j][2] = __ldg(p + 2);
      nxs[j] = ok ? __ldg(up + static_cast<size_t>(s) * MM + mu) : 0.0;
    }
  };
  for (int q = q0; q < q1; ++q) {
    bool own_s = true;
    if constexpr (DIST) {
      const int sq = far_b[q];
      own_s = owned[sq] != 0;
      if (own_s && sq < t) continue;  // warp-uniform
    }
    double sx[CN][3], xs[CN], ps[CN];
    load(q);
#pragma unroll
    for (int j = 0; j < CN; ++j) {
      sx[j][0] = nsx[j][0];
      sx[j][1] = nsx[j][1];
      sx[j][2] = nsx[j][2];
      xs[j] = nxs[j];
      ps[j] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < RN; ++i)
#pragma unroll
      for (int j = 0; j < CN; ++j) {
        const double d0 = tx[i][0] - sx[j][0], d1 = tx[i][1] - sx[j][1], d2 = tx[i][2] - sx[j][2];
        const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
        const double gk = far_rsqrt(r2);  // kFarScale * 4 pi G
        acc[i] = fma(gk, xs[j], acc[i]);
        ps[j] = fma(gk, xt[i], ps[j]);
      }
    if (DIST && !own_s) continue;  // one-sided pair: no transposed product
    // K^T up[t] for the CN columns: reduce over the BR lanes of the column
#pragma unroll
    for (int j = 0; j < CN; ++j) {
      double v = ps[j];
#pragma unroll
      for (int o = 1; o < BR; o <<= 1) {
        const double w = __shfl_down_sync(0xffffffffu, v, o);
        if (bi + o < BR) v += w;
      }
      ps[j] = v;
    }
    if (act && bi == 0) {
      double* dst = slot + static_cast<size_t>(trans[q]) * MM;
#pragma unroll
      for (int j = 0; j < CN; ++j) {
        const int mu = bj + BC * j;
        if (mu < MM) dst[mu] = ps[j] * kFarScale;
      }
    }
  }
  // K up[s] summed over the warp's sources: reduce over the BC lanes of the row
#pragma unroll
  for (int i = 0; i < RN; ++i) {
    double v = acc[i];
#pragma unroll
    for (int o = 1; o < BC; o <<= 1) {
      const double w = __shfl_down_sync(0xffffffffu, v, o * BR);
      if (bj + o < BC) v += w;
    }
    acc[i] = v;
  }
  if (bj == 0) {
#pragma unroll
    for (int i = 0; i < RN; ++i) {
      const int nu = bi + BR * i;
      if (nu < MM) down[static_cast<size_t>(t) * MM + nu] = acc[i] * kFarScale;
    }
  }
}

template <int M, bool DIST, int MINB>
__global__ void __launch_bounds__(256, MINB) k_far_sym(int n_targets, const int* __restrict__ targets,
                                                 const int* __restrict__ upper_start, const int* __restrict__ far_rs,
                                                 const int* __restrict__ far_b, const int* __restrict__ trans,
                                                 const double* __restrict__ img, const double* __restrict__ up,
                                                 double* __restrict__ down, double* __restrict__ slot,
                                                 const unsigned char* __restrict__ owned, int full_row) {
  far_sym_body<M, DIST>(n_targets, targets, upper_start, far_rs, far_b, trans, img, up, down, slot, owned, full_row);
}
// Column-stream symmetric far field (Laplace, single GPU): warp per target t.
// The source columns of all upper pairs (t, s), s > t, are streamed 32 at a
// time -- lane = one interpolation point mu of one pair, so no lane idles
// whatever m^2 is -- while the target's m^2 rows sit in shared memory and are
// broadcast.  Distances in shifted dot form: with c = img[t][0],
// t' = img[t][nu] - c and s' = img[s][mu] - c,
//   |t - s|^2 = (|t'|^2 + |s'|^2) - 2 t'.s'   (one add + three FMAs),
// which is accurate because |t'| and |s'| are bounded by a small multiple of
// |t - s| on admissible pairs; 2/r from the MUFU estimate + one Newton step.
// Per evaluation 9 FP64 instructions (vs 11 in the lane-tile kernel), and the
// transposed product K^T up[t] is one lane's own column sum (no shuffles): it
// goes straight to the slot of the transposed pair (s, t).  K up[s] is
// accumulated per row in registers and reduced over the warp at the end by a
// reduce-scatter butterfly (lane l ends with row l).
template <int MM>
struct ColRows {
  static constexpr int R = MM <= 4 ? 4 : MM <= 8 ? 8 : MM <= 16 ? 16 : 32;  // rows padded to a power of two
  static_assert(MM <= 32, "column-stream far field: m^2 <= 32");
};
template <int MM>
__device__ __forceinline__ void col_reduce_rows(double (&acc)[ColRows<MM>::R], int lane) {
  constexpr int R = ColRows<MM>::R;
  // lanes l and l ^ o (o >= R) hold the same row set: plain sums first
#pragma unroll
  for (int o = 16; o >= R; o >>= 1)
#pragma unroll
    for (int i = 0; i < R; ++i) acc[i] += __shfl_xor_sync(0xffffffffu, acc[i], o);
  // reduce-scatter: at half-width H the lanes with bit H set keep the upper half
#pragma unroll
  for (int H = R / 2; H >= 1; H >>= 1) {
    const bool hi = (lane & H) != 0;
#pragma unroll
    for (int i = 0; i < H; ++i) {
      const double send = hi ? acc[i] : acc[i + H];
      const double keep = hi ? acc[i + H] : acc[i];
      acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, H);
    }
  }
}

// LIST (multi-GPU ranks): the target's columns come from an explicit pair list
// (col_q[col_rs[w] ..]): q >= 0 a pair with an owned source s > t (symmetric:
// the transposed product goes to the slot of (s, t)), ~q a pair whose source
// is another rank's node (one-sided: no slot; that rank evaluates its own side)
template <int M, int C, bool LIST = false>
__device__ __forceinline__ void far_col_body(int t, int lane, double* __restrict__ sh,
                                             const int* __restrict__ upper_start, const int* __restrict__ far_rs,
                                             const int* __restrict__ far_b, const int* __restrict__ trans,
                                             const double* __restrict__ img, const double* __restrict__ up,
                                             double* __restrict__ down, double* __restrict__ slot,
                                             const int* __restrict__ col_q = nullptr, int col_q0 = 0,
                                             int col_q1 = 0) {
  constexpr int MM = M * M, R = ColRows<MM>::R;
  // target rows: sh[4 nu .. 4 nu + 3] = (-2 t'x, -2 t'y, -2 t'z, |t'|^2) (two
  // 16 B broadcasts), sh[4 MM + nu] = up[t][nu]
  const double* ti = img + static_cast<size_t>(t) * MM * 3;
  const double cx = __ldg(ti), cy = __ldg(ti + 1), cz = __ldg(ti + 2);
  for (int nu = lane; nu < MM; nu += 32) {
    const double x = __ldg(ti + 3 * nu) - cx, y = __ldg(ti + 3 * nu + 1) - cy, z = __ldg(ti + 3 * nu + 2) - cz;
    double* r = sh + 4 * nu;
    r[0] = -2.0 * x;
    r[1] = -2.0 * y;
    r[2] = -2.0 * z;
    r[3] = x * x + y * y + z * z;
    sh[4 * MM + nu] = __ldg(up + static_cast<size_t>(t) * MM + nu);
  }
  __syncwarp();
  double acc[R];
#pragma unroll
  for (int i = 0; i < R; ++i) acc[i] = 0.0;
  const int q0 = LIST ? col_q0 : upper_start[t];
  const int ncol = ((LIST ? col_q1 : far_rs[t + 1]) - q0) * MM;
  // the source node of column c (and its pair): read one chunk ahead, so the
  // chunk's point loads depend on registers, not on loads of the same chunk
  auto col_src = [&](int c, int& q, bool& sym) -> int {
    const int qi = c / MM;
    if constexpr (LIST) {
      const int qe = __ldg(col_q + q0 + qi);
      sym = qe >= 0;
      q = qe >= 0 ? qe : ~qe;
    } else {
      sym = true;
      q = q0 + qi;
    }
    return __ldg(far_b + q);
  };
  int s_nx[C], q_nx[C];
  bool sym_nx[C];
#pragma unroll
  for (int k = 0; k < C; ++k) {
    const int c = 32 * k + lane;
    s_nx[k] = c < ncol ? col_src(c, q_nx[k], sym_nx[k]) : t;
  }
  // C columns per lane: each broadcast target row feeds C evaluations
  for (int c0 = 0; c0 < ncol; c0 += 32 * C) {
    double sx[C], sy[C], sz[C], xs[C], ns[C], ps[C];
    int q[C], mu[C];
    bool ok[C], sym[C];
#pragma unroll
    for (int k = 0; k < C; ++k) {
      const int c = c0 + 32 * k + lane;
      ok[k] = c < ncol;
      mu[k] = ok[k] ? c - (c / MM) * MM : 0;
      q[k] = q_nx[k];
      sym[k] = sym_nx[k];
      const int s = s_nx[k];
      const int cn = c + 32 * C;
      s_nx[k] = cn < ncol ? col_src(cn, q_nx[k], sym_nx[k]) : t;
      const double* p = img + (static_cast<size_t>(s) * MM + mu[k]) * 3;
      sx[k] = __ldg(p) - cx;
      sy[k] = __ldg(p + 1) - cy;
      sz[k] = __ldg(p + 2) - cz;
      xs[k] = __ldg(up + static_cast<size_t>(s) * MM + mu[k]);
      if (!ok[k]) {  // padding column: far away (finite kernel), zero weight
        sx[k] = 1.0e8;
        sy[k] = sz[k] = 0.0;
        xs[k] = 0.0;
      }
      ns[k] = sx[k] * sx[k] + sy[k] * sy[k] + sz[k] * sz[k];
      ps[k] = 0.0;
    }
#pragma unroll
    for (int nu = 0; nu < MM; ++nu) {
      const double2 a01 = *reinterpret_cast<const double2*>(sh + 4 * nu);
      const double2 a23 = *reinterpret_cast<const double2*>(sh + 4 * nu + 2);
      const double xt = sh[4 * MM + nu];
#pragma unroll
      for (int k = 0; k < C; ++k) {
        const double r2 = fma(a01.x, sx[k], fma(a01.y, sy[k], fma(a23.x, sz[k], a23.y + ns[k])));
        const double gk = far_rsqrt(r2);  // kFarScale * 4 pi G
        acc[nu] = fma(gk, xs[k], acc[nu]);
        ps[k] = fma(gk, xt, ps[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < C; ++k)
      if (ok[k] && sym[k]) slot[static_cast<size_t>(__ldg(trans + q[k])) * MM + mu[k]] = ps[k] * kFarScale;
  }
  col_reduce_rows<MM>(acc, lane);
  if (lane < MM) down[static_cast<size_t>(t) * MM + lane] = acc[0] * kFarScale;
}

template <int M, int MINB, int C>
__global__ void __launch_bounds__(256, MINB) k_far_col(int n_targets, const int* __restrict__ targets,
                                                      const int* __restrict__ upper_start,
                                                      const int* __restrict__ far_rs, const int* __restrict__ far_b,
                                                      const int* __restrict__ trans, const double* __restrict__ img,
                                                      const double* __restrict__ up, double* __restrict__ down,
                                                      double* __restrict__ slot) {
  __shared__ __align__(16) double sh[8][(5 * M * M + 1) / 2 * 2];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_targets) return;
  far_col_body<M, C>(targets[warp], threadIdx.x & 31, sh[threadIdx.x >> 5], upper_start, far_rs, far_b, trans, img,
                     up, down, slot);
}

template <int M, int MINB, int C>
__global__ void __launch_bounds__(256, MINB) k_far_col_list(int n_targets, const int* __restrict__ targets,
                                                           const int* __restrict__ col_rs, const int* __restrict__ col_q,
                                                           const int* __restrict__ far_b, const int* __restrict__ trans,
                                                           const double* __restrict__ img, const double* __restrict__ up,
                                                           double* __restrict__ down, double* __restrict__ slot) {
  __shared__ __align__(16) double sh[8][(5 * M * M + 1) / 2 * 2];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_targets) return;
  far_col_body<M, C, true>(targets[warp], threadIdx.x & 31, sh[threadIdx.x >> 5], nullptr, nullptr, far_b, trans, img,
                           up, down, slot, col_q, col_rs[warp], col_rs[warp + 1]);
}

// down[s] += sum of the transposed contributions of the pairs (s, t), t < s,
// in ascending t (fixed order)
// Unconditional, unrolled stream over the row's contiguous slots.  Multi-GPU:
// only owned rows; the slots of pairs whose other node is another rank's are
// never written and stay zero from construction.
// rows: 0 all, 1 leaf-level rows only, 2 the other levels (level-split graph)
template <bool DIST>
__global__ void k_far_lower(int n_nodes, int mm, const int* __restrict__ far_rs, const int* __restrict__ upper_start,
                            const int* __restrict__ far_b, const unsigned char* __restrict__ owned,
                            const double* __restrict__ slot, double* __restrict__ down, int rows = 0, int npp = 1,
                            int leaf_off = 0) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_nodes) * mm) return;
  const int s = static_cast<int>(idx / mm), nu = static_cast<int>(idx % mm);
  if (rows != 0 && ((s % npp >= leaf_off) != (rows == 1))) return;
  const int q0 = far_rs[s], q1 = upper_start[s];
  if (q0 == q1 || (DIST && !owned[s])) return;
  double acc = down[idx];
  const double* sp = slot + static_cast<size_t>(q0) * mm + nu;
  (void)far_b;
#pragma unroll 8
  for (int q = q0; q < q1; ++q, sp += mm) acc += __ldcs(sp);  // read once: streaming
  down[idx] = acc;
}

// child(i,j) += tu^T X tv  (h2.cpp:328-347): children at level+1 >= 1 in
// level-1 clusters [c0, c1); M as in k_up_level
template <class S, int M>
__global__ void k_down_level(int np, int level, int npp, int off_p, int off_c, int m_rt, int nch,
                             const double* __restrict__ tl, const double* __restrict__ tr, S* __restrict__ down,
                             int c0, int c1) {
  pdl_entry();
  (void)np;
  const int m = M ? M : m_rt;
  const int mm = m * m, rows = nch * mm, cside = 2 << level, per = 1 << (2 * level);
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(c1 - c0) * per * rows) return;
  const int r = static_cast<int>(idx % rows);
  const long long nidx = idx / rows;
  int p, sx, sy;
  cluster_node(c0 + static_cast<int>(nidx / per), level + 1, static_cast<int>(nidx % per), p, sx, sy);
  const int c = r / mm, nu = r % mm, i = nu % m, j = nu / m;
  const int parent = p * npp + off_p + (sx / 2) + (cside / 2) * (sy / 2);
  const double* tu = (sx & 1) ? tr : tl;
  const double* tv = (sy & 1) ? tr : tl;
  const S* X = down + static_cast<size_t>(parent) * rows + c * mm;
  S acc = zero<S>();
#pragma unroll
  for (int b = 0; b < m; ++b) {
    S t = zero<S>();
#pragma unroll
    for (int a = 0; a < m; ++a) fmac(t, X[a + m * b], __ldg(tu + a + m * i));
    fmac(acc, t, __ldg(tv + b + m * j));
  }
  S* Y = down + static_cast<size_t>(p * npp + off_c + sx + cside * sy) * rows + c * mm;
  Y[nu] = Y[nu] + acc;
}

// all-gather payload of the up moments (owned nodes, levels >= 1)
template <class S>
__global__ void k_pack(int n, const int* __restrict__ nodes, int rows, const S* __restrict__ up, S* __restrict__ send) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n) * rows) return;
  send[idx] = up[static_cast<size_t>(nodes[idx / rows]) * rows + idx % rows];
}
template <class S>
__global__ void k_unpack(int n, const int* __restrict__ nodes, int rows, const S* __restrict__ recv, S* __restrict__ up) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n) * rows) return;
  const int node = nodes[idx / rows];
  if (node >= 0) up[static_cast<size_t>(node) * rows + idx % rows] = recv[idx];
}

// near-field rows per test element (h2.cpp:349-357); one warp per element,
// streaming its contiguous row [la][k][lb]
// FROM_X: coefficients gathered inline from x (l2g, signs) instead of coef
template <class S, int NL, bool FROM_X>
__device__ __forceinline__ void near_row(int e, int lane, const int* __restrict__ near_rs,
                                         const int* __restrict__ near_b, const S* __restrict__ blk,
                                         const S* __restrict__ coef, S* __restrict__ rows_out,
                                         const int* __restrict__ l2g, const double* __restrict__ sg) {
  auto cf = [&](int k) -> S {
    if constexpr (FROM_X) return coef[l2g[k]] * sg[k];
    else return coef[k];
  };
  const int rs = near_rs[e], cnt = near_rs[e + 1] - rs;
  const int len = cnt * NL;
  const S* base = blk + static_cast<size_t>(rs) * NL * NL;
  S acc[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) acc[l] = zero<S>();
  constexpr int U = (NL <= 9) ? 4 : 2;
  int j = lane;
  for (; j + 32 * (U - 1) < len; j += 32 * U) {
    S xv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int jj = j + 32 * u, k = jj / NL, lb = jj - k * NL;
      xv[u] = cf(near_b[rs + k] * NL + lb);
    }
#pragma unroll
    for (int la = 0; la < NL; ++la)
#pragma unroll
      for (int u = 0; u < U; ++u) fmac(acc[la], ldg_s(base + static_cast<size_t>(la) * len + j + 32 * u), xv[u]);
  }
  for (; j < len; j += 32) {
    const int k = j / NL, lb = j - k * NL;
    const S xv = cf(near_b[rs + k] * NL + lb);
#pragma unroll
    for (int la = 0; la < NL; ++la) fmac(acc[la], ldg_s(base + static_cast<size_t>(la) * len + j), xv);
  }
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const S a = warp_sum(acc[l]);
    if (lane == 0) rows_out[static_cast<size_t>(e) * NL + l] = a;
  }
}
template <class S, int NL, bool FROM_X = false>
__global__ void __launch_bounds__(256) k_near_rows(int ne, const int* __restrict__ near_rs,
                                                   const int* __restrict__ near_b, const S* __restrict__ blk,
                                                   const S* __restrict__ coef, S* __restrict__ rows_out,
                                                   const int* __restrict__ l2g = nullptr,
                                                   const double* __restrict__ sg = nullptr) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= ne) return;
  near_row<S, NL, FROM_X>(e, threadIdx.x & 31, near_rs, near_b, blk, coef, rows_out, l2g, sg);
}

// Leaf-level column-stream far field fused with the near rows (single GPU): as
// the HBM-bound rows run at the tail of each warp while other warps of the SM
// are still in the FP64-bound far loop.
template <int M, int NL, int MINB, int C>
__global__ void __launch_bounds__(256, MINB) k_far_col_near(
    int n_fine, const int* __restrict__ fine, int n_rest, const int* __restrict__ rest, int epp, int npp,
    int leaf_off, const int* __restrict__ upper_start, const int* __restrict__ far_rs,
    const int* __restrict__ far_b, const int* __restrict__ trans, const double* __restrict__ img,
    const double* __restrict__ up, double* __restrict__ down, double* __restrict__ slot,
    const unsigned char* __restrict__ /*owned: single GPU*/, const int* __restrict__ near_rs,
    const int* __restrict__ near_b, const double* __restrict__ blk, const double* __restrict__ x,
    double* __restrict__ rows_out, const int* __restrict__ l2g, const double* __restrict__ sg) {
  __shared__ __align__(16) double sh[8][(5 * M * M + 1) / 2 * 2];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int e;
  if (warp < n_fine) {
    const int t = fine[warp];
    far_col_body<M, C>(t, lane, sh[threadIdx.x >> 5], upper_start, far_rs, far_b, trans, img, up, down, slot);
    e = (t / npp) * epp + (t % npp - leaf_off);
  } else if (warp < n_fine + n_rest) {
    e = rest[warp - n_fine];
  } else {
    return;
  }
  near_row<double, NL, true>(e, lane, near_rs, near_b, blk, x, rows_out, l2g, sg);
}

// leaf backward transform moments^T down + near rows (h2.cpp:359-371); one
// thread per (owned element, local function)
template <class S, int NL>
__global__ void __launch_bounds__(256) k_leaf_down(int n_el, const int* __restrict__ el, int rows, int epp, int npp,
                                                   int leaf_off, const double* __restrict__ mom,
                                                   const S* __restrict__ down, const S* __restrict__ near_rows,
                                                   S* __restrict__ loc) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_el) * NL) return;
  const int i = static_cast<int>(idx / NL), l = static_cast<int>(idx % NL);
  const int e = el[i];
  const int leaf = (e / epp) * npp + leaf_off + (e % epp);
  const S* dn = down + static_cast<size_t>(leaf) * rows;
  const double* mc = mom + (static_cast<size_t>(e) * NL + l) * rows;
  S acc = zero<S>();
  if constexpr (sizeof(S) == 8) {
    // rows even (m^2 nch with m even or nch = 4) and 16 B aligned: paired loads
    if ((rows & 1) == 0) {
      const double2* m2 = reinterpret_cast<const double2*>(mc);
      const double2* d2 = reinterpret_cast<const double2*>(dn);
#pragma unroll 8
      for (int r = 0; r < rows / 2; ++r) {
        const double2 a = __ldg(m2 + r), b = d2[r];
        acc = fma(b.x, a.x, acc);
        acc = fma(b.y, a.y, acc);
      }
      loc[idx] = near_rows[idx] + acc;
      return;
    }
  }
#pragma unroll 8
  for (int r = 0; r < rows; ++r) fmac(acc, dn[r], __ldg(mc + r));
  loc[idx] = near_rows[idx] + acc;
}

template <class S>
__global__ void k_scatter(int nd, const int* __restrict__ start, const int* __restrict__ inc,
                          const double* __restrict__ sg, const S* __restrict__ loc, S* __restrict__ y) {
  pdl_entry();
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  S acc = zero<S>();
  for (int i = start[d]; i < start[d + 1]; ++i) {
    const int k = inc[i];
    acc = acc + loc[k] * sg[k];
  }
  y[d] = acc;
}

template <class S>
__global__ void k_zero(size_t n, S* p) {
  pdl_entry();
  const size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x;
  if (i < n) p[i] = zero<S>();
}

}  // namespace dev

// ====================================================== host driver
using namespace dev;

// Small, latency-bound kernels of the matvec chains are launched with
// programmatic stream serialisation: a launch may become resident while its
// predecessor finishes (each such kernel begins with pdl_entry()).
template <class... KArgs, class... Args>
static void pdl_launch(void (*kern)(KArgs...), unsigned grid, unsigned block, size_t smem, cudaStream_t s,
                       Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1 ? 1 : 0;
  IGB_CUDA(cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...));
}

// transfer kernels with the interpolation degree as a template parameter
template <class S, class... A>
static void launch_up_level(unsigned grid, cudaStream_t s, A... a) {
  const int m = std::get<5>(std::make_tuple(a...));
  switch (m) {
    case 2: pdl_launch(k_up_level<S, 2>, grid, 256, 0, s, a...); break;
    case 3: pdl_launch(k_up_level<S, 3>, grid, 256, 0, s, a...); break;
    case 4: pdl_launch(k_up_level<S, 4>, grid, 256, 0, s, a...); break;
    case 5: pdl_launch(k_up_level<S, 5>, grid, 256, 0, s, a...); break;
    case 6: pdl_launch(k_up_level<S, 6>, grid, 256, 0, s, a...); break;
    case 7: pdl_launch(k_up_level<S, 7>, grid, 256, 0, s, a...); break;
    case 8: pdl_launch(k_up_level<S, 8>, grid, 256, 0, s, a...); break;
    default: pdl_launch(k_up_level<S, 0>, grid, 256, 0, s, a...); break;
  }
}
template <class S, class... A>
static void launch_down_level(unsigned grid, cudaStream_t s, A... a) {
  const int m = std::get<5>(std::make_tuple(a...));
  switch (m) {
    case 2: pdl_launch(k_down_level<S, 2>, grid, 256, 0, s, a...); break;
    case 3: pdl_launch(k_down_level<S, 3>, grid, 256, 0, s, a...); break;
    case 4: pdl_launch(k_down_level<S, 4>, grid, 256, 0, s, a...); break;
    case 5: pdl_launch(k_down_level<S, 5>, grid, 256, 0, s, a...); break;
    case 6: pdl_launch(k_down_level<S, 6>, grid, 256, 0, s, a...); break;
    case 7: pdl_launch(k_down_level<S, 7>, grid, 256, 0, s, a...); break;
    case 8: pdl_launch(k_down_level<S, 8>, grid, 256, 0, s, a...); break;
    default: pdl_launch(k_down_level<S, 0>, grid, 256, 0, s, a...); break;
  }
}

// Device memory comes from one stream-ordered pool per device that keeps
// freed memory reserved (release threshold = max): operators built and
// destroyed repeatedly -- a solve per right-hand side / geometry -- reuse it
// instead of paying the driver's map / unmap on every construction.
static cudaMemPool_t device_pool(int device) {
  static std::mutex mu;
  static std::map<int, cudaMemPool_t> pools;
  std::lock_guard<std::mutex> lock(mu);
  auto it = pools.find(device);
  if (it != pools.end()) return it->second;
  cudaMemPoolProps props = {};
  props.allocType = cudaMemAllocationTypePinned;
  props.location.type = cudaMemLocationTypeDevice;
  props.location.id = device;
  cudaMemPool_t pool;
  IGB_CUDA(cudaMemPoolCreate(&pool, &props));
  // IGB_POOL_KEEP_MB bounds what stays reserved between operators (default:
  // everything); igb_release_device_memory() trims it on demand
  uint64_t keep = UINT64_MAX;
  if (const char* e = std::getenv("IGB_POOL_KEEP_MB")) keep = std::strtoull(e, nullptr, 10) << 20;
  IGB_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  pools[device] = pool;
  return pool;
}

void release_device_memory(int device) {
  cudaMemPool_t pool = device_pool(device);
  IGB_CUDA(cudaSetDevice(device));
  IGB_CUDA(cudaDeviceSynchronize());
  IGB_CUDA(cudaMemPoolTrimTo(pool, 0));
}

// Pinned host staging buffers of the host-vector apply, recycled across
// operators (cudaMallocHost costs milliseconds).
static std::mutex g_pinned_mu;
static std::multimap<size_t, void*> g_pinned_free;
static std::map<void*, size_t>& g_pinned_sizes() {
  static std::map<void*, size_t> m;
  return m;
}
static void pinned_put(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lock(g_pinned_mu);
  g_pinned_free.emplace(g_pinned_sizes()[p], p);
}
static void* pinned_get(size_t bytes) {
  {
    std::lock_guard<std::mutex> lock(g_pinned_mu);
    auto it = g_pinned_free.lower_bound(bytes);
    if (it != g_pinned_free.end() && it->first <= 2 * bytes) {
      void* p = it->second;
      g_pinned_free.erase(it);
      return p;
    }
  }
  void* p = nullptr;
  IGB_CUDA(cudaMallocHost(&p, bytes));
  std::lock_guard<std::mutex> lock(g_pinned_mu);
  g_pinned_sizes()[p] = bytes;
  return p;
}

template <class T>
T* H2Device::dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  const auto t0 = std::chrono::steady_clock::now();
  cudaStream_t s = up_stream_ ? up_stream_ : stream_;
  const cudaError_t e = cudaMallocFromPoolAsync(&p, n * sizeof(T), device_pool(device_), s);
  if (e == cudaErrorMemoryAllocation) {
    cudaGetLastError();
    throw std::runtime_error("B200 H2: out of device memory (" + std::to_string(n * sizeof(T)) + " bytes)");
  }
  IGB_CUDA(e);
  alloc_ms_ += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  allocs_.push_back(p);
  return static_cast<T*>(p);
}

void H2Device::release_memory() {
  // work on user streams (apply_device) may still read the buffers: the same
  // device-wide wait cudaFree performs, then the stream-ordered frees
  cudaDeviceSynchronize();
  for (void* p : allocs_) cudaFreeAsync(p, stream_);
  allocs_.clear();
  cudaStreamSynchronize(stream_);
}
template <class T>
T* H2Device::upload(const std::vector<T>& v) {
  T* p = dalloc<T>(v.size());
  upload_bytes_ += v.size() * sizeof(T);
  if (!v.empty())
    IGB_CUDA(cudaMemcpyAsync(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, up_stream_ ? up_stream_ : stream_));
  return p;
}

static unsigned grid_for(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

H2Device::H2Device(std::shared_ptr<const Discretization> d, int m, double eta, int far_order, int sing_order,
                   int device, int flags, int world, int rank)
    : disc_(std::move(d)), device_(device), flags_(flags) {
  if (world < 1 || rank < 0 || rank >= world) throw std::invalid_argument("H2Matrix: bad rank/world");
  if (world > 1 && (flags & kStoredCouplings))
    throw std::invalid_argument("H2Matrix: stored couplings are single-GPU only");
  if ((flags & kStoredCouplings) && (flags & kFusedCouplings))
    throw std::invalid_argument("H2Matrix: stored and on-the-fly couplings requested together");
  const auto t_wall0 = std::chrono::steady_clock::now();
  check_h2_options(*disc_, m, eta, far_order, sing_order, &nfar_, &nsing_);
  if (nsing_ > 16) throw std::invalid_argument("B200 H2: singular order > 16 not supported (32-bit point index)");
  opt_ = {m, eta, far_order, sing_order, world, rank};
  int ndev = 0;
  IGB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw std::invalid_argument("H2Matrix: CUDA device index out of range");
  IGB_CUDA(cudaSetDevice(device_));
  IGB_CUDA(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
  IGB_CUDA(cudaStreamCreateWithFlags(&aux_, cudaStreamNonBlocking));
  nch_ = disc_->is_vector() ? 4 : 1;
  {
    const int q = disc_->kind() == kMaxwell ? disc_->degree() : disc_->scalar_degree();
    if (disc_->kind() == kMaxwell && (q < 1 || q > 3))
      throw std::invalid_argument("B200 H2: Maxwell degree > 3 not instantiated");
    if (disc_->kind() != kMaxwell && (q < 0 || q > 4))
      throw std::invalid_argument("B200 H2: scalar space degree > 4 not instantiated");
  }
  try {
    dispatch_kind([&](auto kt) { assemble_impl<decltype(kt)>(t_wall0); });
  } catch (...) {
    cudaStreamSynchronize(aux_);
    release_memory();
    cudaStreamDestroy(aux_);
    cudaStreamDestroy(stream_);
    aux_ = stream_ = nullptr;
    throw;
  }
  times_.total_wall = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count();
}

H2Device::~H2Device() {
  cudaSetDevice(device_);
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph1_) cudaGraphExecDestroy(graph1_);
  if (graph2_) cudaGraphExecDestroy(graph2_);
  release_memory();
  pinned_put(h_x_pinned_);
  pinned_put(h_y_pinned_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (ev_fork2_) cudaEventDestroy(ev_fork2_);
  if (ev_join2_) cudaEventDestroy(ev_join2_);
  if (ev_apply_done_) cudaEventDestroy(ev_apply_done_);
  if (side_) cudaStreamDestroy(side_);
  if (side2_) cudaStreamDestroy(side2_);
  if (aux_) cudaStreamDestroy(aux_);
  if (stream_) cudaStreamDestroy(stream_);
}

// Construction is a two-stage pipeline.  Stage 1 needs only the mesh: the
// element caches / moments and the singular integrals (the bulk of the device
// work) are launched before the block partition exists -- the singular items
// come from the mesh topology (Discretization::singular_items).  Stage 2 builds
// the block partition on the host while the device integrates, uploads it on a
// second stream, and launches images, regular near blocks and the scatter of
// the singular blocks into their near slots.
template <class KT>
void H2Device::assemble_impl(std::chrono::steady_clock::time_point t_wall0) {
  const Discretization& d = *disc_;
  static const bool verbose = getenv("IGB_VERBOSE") != nullptr;
  auto lap = [&](const char* what) {
    if (verbose)
      fprintf(stderr, "[igb ctor] %-16s %8.2f ms\n", what,
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_wall0).count());
  };
  if (d.local_count() != KT::NL) throw std::logic_error("B200 H2: local count mismatch");
  // ---- stage 1: mesh-only data and kernels
  std::vector<unsigned char> owned;
  if (opt_.world > 1) owned = owned_elements(d, opt_.world, opt_.rank);
  d.singular_items(owned.empty() ? nullptr : owned.data(), sing_items_);
  lap("singular items");
  auto tu = std::chrono::steady_clock::now();
  stage_elements<KT>();
  double up_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tu).count();
  cudaEvent_t ev[kAsmEvents];
  for (auto& e : ev) IGB_CUDA(cudaEventCreate(&e));
  int launched = 0;
  IGB_CUDA(cudaEventRecord(ev[0], stream_));
  launch_element_phase<KT>(ev, launched);
  lap("stage 1 launched");
  // ---- stage 2: block partition on the host, overlapping the device
  const auto t0 = std::chrono::steady_clock::now();
  plan_ = build_plan(d, opt_.m, opt_.eta, opt_.far_order, opt_.sing_order, (flags_ & 4) ? device_ : -1);
  lp_ = build_local_plan(d, plan_, opt_.world, opt_.rank);
  times_.plan_host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  lap("plan");
  // couplings stored or evaluated in every matvec: unless forced, complex kinds
  // store them when they fit in half the free device memory -- their m^4
  // complex kernel evaluations per pair cost more than streaming the block
  // (c4: 6.2 ms per matvec stored at 93 % of HBM vs 14.6 ms evaluated); Laplace
  // always evaluates them (c5: the symmetric FP64 kernel beats the 161 GB stream)
  if (!(flags_ & (kStoredCouplings | kFusedCouplings)) && opt_.world == 1 && d.is_complex()) {
    size_t free_b = 0, total_b = 0;
    IGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
    const size_t mm = static_cast<size_t>(opt_.m) * opt_.m;
    if (plan_.far_a.size() * mm * mm * 16 <= free_b / 2) flags_ |= kStoredCouplings;
  }
  for (int c = 1; c <= 3; ++c) {  // topology items == the near list's singular pairs
    const SingList &T = sing_items_[c], &L = lp_.sing[c];
    if (T.ea != L.ea || T.eb != L.eb || T.map_a != L.map_a || T.map_b != L.map_b)
      throw std::logic_error("B200 H2: singular pairs of the mesh topology differ from the near field");
  }
  tu = std::chrono::steady_clock::now();
  up_stream_ = aux_;
  alloc_ms_ = 0;
  stage_plan<KT>();
  up_stream_ = nullptr;
  if (verbose) fprintf(stderr, "[igb ctor] stage-2 cudaMalloc total %.2f ms\n", alloc_ms_);
  up_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tu).count();
  times_.upload = up_ms;
  IGB_CUDA(cudaEventRecord(ev[kEvUploaded], aux_));
  IGB_CUDA(cudaStreamWaitEvent(stream_, ev[kEvUploaded], 0));
  lap("stage 2 uploaded");
  IGB_CUDA(cudaEventRecord(ev[kEvPlanPhase], stream_));
  launch_plan_phase<KT>(ev, launched);
  IGB_CUDA(cudaStreamSynchronize(stream_));
  collect_times(ev);
  for (auto& e : ev) cudaEventDestroy(e);
  ++assembly_launches_count_;
  assembly_kernels_ = launched;
  lap("assembled");
  alloc_ms_ = 0;
  // ---- matvec scratch
  const H2Plan& P = plan_;
  const LocalPlan& Lp = lp_;
  const int ne = d.element_count(), m = P.m, mm = m * m, rows = nch_ * mm, NL = KT::NL;
  const int sw = sizeof(typename KT::S) / 8;
  const size_t nn = static_cast<size_t>(P.n_nodes);
  dx_ = dalloc<double>(static_cast<size_t>(d.dof_count()) * sw);
  dy_ = dalloc<double>(static_cast<size_t>(d.dof_count()) * sw);
  d_coef_ = dalloc<double>(static_cast<size_t>(ne) * NL * sw);
  if (Lp.world > 1) {
    d_send_ = dalloc<double>(static_cast<size_t>(Lp.pack_max) * rows * sw);
    d_recv_ = dalloc<double>(static_cast<size_t>(Lp.pack_max) * Lp.world * rows * sw);
  }
  d_up_ = dalloc<double>(nn * rows * sw);
  d_down_ = dalloc<double>(nn * rows * sw);
  d_loc_ = dalloc<double>(Lp.el.size() * NL * sw);
  d_nrows_ = dalloc<double>(Lp.el.size() * NL * sw);
  IGB_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  IGB_CUDA(cudaStreamCreateWithFlags(&side2_, cudaStreamNonBlocking));
  IGB_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  IGB_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  IGB_CUDA(cudaEventCreateWithFlags(&ev_fork2_, cudaEventDisableTiming));
  IGB_CUDA(cudaEventCreateWithFlags(&ev_join2_, cudaEventDisableTiming));
  IGB_CUDA(cudaEventCreateWithFlags(&ev_apply_done_, cudaEventDisableTiming));
  IGB_CUDA(cudaEventRecord(ev_apply_done_, stream_));
  IGB_CUDA(cudaMemsetAsync(d_up_, 0, nn * rows * sw * 8, stream_));
  IGB_CUDA(cudaFuncSetAttribute(k_far_cta<typename KT::S, 4, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_cta<typename KT::S, 1, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_fused<KT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_fused<KT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_fused<KT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_sym_w<KT, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_sym_w<KT, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_sym_w<KT, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaFuncSetAttribute(k_far_sym_w<KT, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  IGB_CUDA(cudaStreamSynchronize(stream_));
  if (verbose) fprintf(stderr, "[igb ctor] scratch cudaMalloc total %.2f ms\n", alloc_ms_);
  lap("scratch");
}

// Stage-1 inputs: geometry cells, basis tables, DOF maps, quadrature rules and
// the singular work lists; element-phase outputs.
template <class KT>
void H2Device::stage_elements() {
  const Discretization& d = *disc_;
  constexpr int NL = KT::NL, NC = KT::NC;
  const int ne = d.element_count(), m = opt_.m, mm = m * m, rows = nch_ * mm;
  const int sw = sizeof(typename KT::S) / 8;
  std::vector<double> cells(d.cells().size() * kCellStride, 0.0);
  for (size_t c = 0; c < d.cells().size(); ++c) {
    const GeomCell& gc = d.cells()[c];
    for (int comp = 0; comp < 4; ++comp)
      for (int j = 0; j <= kMaxGeomDeg; ++j)
        for (int i = 0; i <= kMaxGeomDeg; ++i) cells[c * kCellStride + comp * 25 + j * 5 + i] = gc.coef[comp][j][i];
    cells[c * kCellStride + 100] = gc.u0;
    cells[c * kCellStride + 101] = gc.v0;
  }
  d_cells_ = upload(cells);
  d_el_cell_ = upload(d.element_cell());
  {
    std::vector<int> info;
    std::vector<double> knots;
    int base = 0;
    for (int p = 0; p < d.geometry().patch_count(); ++p) {
      const Patch& s = d.geometry().patch(p);
      const int ku_off = static_cast<int>(knots.size());
      knots.insert(knots.end(), s.kv_u.knots.begin(), s.kv_u.knots.end());
      const int kv_off = static_cast<int>(knots.size());
      knots.insert(knots.end(), s.kv_v.knots.begin(), s.kv_v.knots.end());
      info.insert(info.end(), {base, s.kv_u.degree, s.kv_v.degree, static_cast<int>(s.kv_u.knots.size()),
                               static_cast<int>(s.kv_v.knots.size()), ku_off, kv_off});
      base += (s.kv_u.size() - s.kv_u.degree) * (s.kv_v.size() - s.kv_v.degree);
    }
    d_patch_info_ = upload(info);
    d_knots_ = upload(knots);
  }
  d_tab_a_ = upload(d.is_vector() ? d.tab_p() : d.tab_s());
  d_tab_b_ = upload(d.is_vector() ? d.tab_q() : std::vector<double>(1, 0.0));
  d_l2g_ = upload(d.l2g());
  d_lsign_ = upload(d.lsign());
  std::vector<double> gxf, gwf, gxs, gws;
  gauss_rule(nfar_, gxf, gwf);
  gauss_rule(nsing_, gxs, gws);
  as_.gxf = upload(gxf);
  as_.gwf = upload(gwf);
  as_.gxs = upload(gxs);
  as_.gws = upload(gws);
  const std::vector<double> cheb = cheb_nodes(m);
  as_.cheb = upload(cheb);
  std::vector<double> lag(static_cast<size_t>(m) * nfar_);
  {
    std::vector<double> tmp(m);
    for (int a = 0; a < nfar_; ++a) {
      lagrange_all(cheb, gxf[a], tmp.data());
      for (int i = 0; i < m; ++i) lag[i * nfar_ + a] = tmp[i];
    }
  }
  as_.lag = upload(lag);
  for (int c = 1; c <= 3; ++c) {
    const SingList& L = sing_items_[c];
    as_.sing[c][0] = upload(L.ea);
    as_.sing[c][1] = upload(L.eb);
    as_.singm[c][0] = upload(L.map_a);
    as_.singm[c][1] = upload(L.map_b);
    d_sing_blk_[c] = dalloc<double>(L.ea.size() * NL * NL * sw);
  }
  const cplx kap = d.kappa();
  as_.kp[0] = kap.real();
  as_.kp[1] = kap.imag();
  if (d.is_vector()) {
    const cplx dw = -1.0 / (kap * kap);
    as_.kp[2] = dw.real();
    as_.kp[3] = dw.imag();
  }
  const int nq = nfar_ * nfar_;
  d_mom_ = dalloc<double>(static_cast<size_t>(ne) * NL * rows);
  d_cpts_ = dalloc<double>(static_cast<size_t>(ne) * nq * 3);
  d_cval_ = dalloc<double>(static_cast<size_t>(ne) * NC * nq * NL);
  bytes_.moments = static_cast<size_t>(ne) * NL * rows * 8;
}

// Stage-2 inputs: the block partition (near / far lists, tree, transfers, DOF
// gather) and the partition-sized outputs.
template <class KT>
void H2Device::stage_plan() {
  const Discretization& d = *disc_;
  const H2Plan& P = plan_;
  const LocalPlan& Lp = lp_;
  constexpr int NL = KT::NL;
  const int m = P.m, mm = m * m;
  const int sw = sizeof(typename KT::S) / 8;
  d_near_a_ = upload(Lp.near_row);  // local row of each local near slot
  d_near_b_ = upload(Lp.near_eb);
  d_near_ea_ = upload(Lp.near_ea);
  d_near_rs_ = upload(Lp.near_rs);
  d_el_ = upload(Lp.el);
  d_owned_ = upload(Lp.node_owned);
  {
    std::vector<double> sg(Lp.el.size() * static_cast<size_t>(d.local_count()));
    for (size_t i = 0; i < Lp.el.size(); ++i)
      for (int l = 0; l < d.local_count(); ++l)
        sg[i * d.local_count() + l] = d.lsign()[static_cast<size_t>(Lp.el[i]) * d.local_count() + l];
    d_loc_sign_ = upload(sg);
  }
  if (Lp.world > 1) {
    d_pack_nodes_ = upload(Lp.pack_nodes);
    std::vector<int> un(static_cast<size_t>(Lp.world) * Lp.pack_max, -1);
    for (int r = 0; r < Lp.world; ++r)
      for (size_t i = 0; i < Lp.rank_pack_nodes[r].size(); ++i) un[static_cast<size_t>(r) * Lp.pack_max + i] = Lp.rank_pack_nodes[r][i];
    d_unpack_nodes_ = upload(un);
  }
  if (stored_couplings()) d_far_a_ = upload(P.far_a);  // only the stored-coupling kernel reads pair rows
  d_far_b_ = upload(P.far_b);
  d_far_rs_ = upload(P.far_row_start);
  {
    const std::vector<int>& targets = Lp.far_targets;
    n_far_targets_ = static_cast<int>(targets.size());
    d_far_targets_ = upload(targets);
    // symmetric fused far field (Laplace, m <= 6): upper pairs + transposes
    sym_far_ = !stored_couplings() && d.kind() == kLaplace && m >= 2 && m <= 6;
    // m <= 5, one GPU: the column-stream kernel, two columns per lane (c5:
    // 14.57 -> 11.0 ms per matvec, c2: 0.379 -> 0.348 ms against the lane-tile
    // kernel, which m = 6 keeps)
    far_col_ = sym_far_ && m <= 5 && Lp.world == 1;
    // other kinds / larger m, one GPU: the warp-row symmetric kernel
    sym_w_ = !stored_couplings() && !sym_far_ && Lp.world == 1 && mm >= 32 && mm <= 128;
    if (sym_far_ || sym_w_) {
      std::vector<int> sym_targets;
      for (int t : Lp.far_targets)
        if (Lp.world > 1 || P.far_upper_start[t] < P.far_row_start[t + 1]) sym_targets.push_back(t);
      // longest rows first (one warp per target): the last wave holds the light
      // rows.  The lane-tile kernel (little work per pair) only while the
      // source data (node images + moments) sits in L2: beyond that node order
      // keeps neighbouring targets, which share source clusters, in
      // neighbouring warps (c5: 15.1 vs 16.7 ms per far field); the warp-row
      // kernel (m^4 complex evaluations per pair) always (c3: 82.9 vs 85.5 ms)
      const double src_bytes = static_cast<double>(P.n_nodes) * mm * (3 + nch_ * sw) * 8.0;
      if (sym_w_ || src_bytes <= 64.0 * (1 << 20)) {
        auto work = [&](int t) {
          return Lp.world > 1 ? P.far_row_start[t + 1] - P.far_row_start[t]
                              : P.far_row_start[t + 1] - P.far_upper_start[t];
        };
        std::stable_sort(sym_targets.begin(), sym_targets.end(), [&](int a, int b) { return work(a) > work(b); });
      }
      n_sym_targets_ = static_cast<int>(sym_targets.size());
      d_sym_targets_ = upload(sym_targets);
      std::vector<int> fine, coarse;
      for (int t : sym_targets) (P.node_level[t] == P.depth ? fine : coarse).push_back(t);
      n_sym_fine_ = static_cast<int>(fine.size());
      n_sym_coarse_ = static_cast<int>(coarse.size());
      for (int t : fine) sym_pairs_[0] += P.far_row_start[t + 1] - P.far_upper_start[t];
      for (int t : coarse) sym_pairs_[1] += P.far_row_start[t + 1] - P.far_upper_start[t];
      d_sym_fine_ = upload(fine);
      d_sym_coarse_ = upload(coarse);
      // fused leaf far field + near rows (single GPU, m = 4): the elements whose
      // leaf has no upper far pairs get near-only warps
      bool ident = Lp.world == 1 && static_cast<int>(Lp.el.size()) == d.element_count();
      for (size_t i = 0; ident && i < Lp.el.size(); ++i) ident = Lp.el[i] == static_cast<int>(i);
      if (far_col_ && (m == 4 || m == 5) && ident) {
        std::vector<char> has(d.element_count(), 0);
        const int epp = d.elements_per_patch();
        for (int t : fine) has[(t / P.npp) * epp + (t % P.npp - P.level_offset[P.depth])] = 1;
        std::vector<int> rest;
        for (int e = 0; e < d.element_count(); ++e)
          if (!has[e]) rest.push_back(e);
        n_near_rest_ = static_cast<int>(rest.size());
        d_near_rest_ = upload(rest);
      }
      if (Lp.world > 1 && sym_far_ && m <= 5) {  // per-target column lists for k_far_col_list
        std::vector<int> col_rs(1, 0), col_q;
        for (int t : sym_targets) {
          for (int q = P.far_row_start[t]; q < P.far_row_start[t + 1]; ++q) {
            const int sq = P.far_b[q];
            if (!Lp.node_owned[sq]) col_q.push_back(~q);
            else if (sq > t) col_q.push_back(q);
          }
          col_rs.push_back(static_cast<int>(col_q.size()));
        }
        d_col_rs_ = upload(col_rs);
        d_col_q_ = upload(col_q);
      }
      d_upper_start_ = upload(P.far_upper_start);
      d_trans_ = upload(P.far_trans);
      const size_t per_pair = static_cast<size_t>(mm) * (sym_w_ ? static_cast<size_t>(nch_) * sw : 1);
      d_slot_ = dalloc<double>(P.far_a.size() * per_pair);
      // slots no kernel writes (multi-GPU: pairs with another rank's node) read as 0
      IGB_CUDA(cudaMemsetAsync(d_slot_, 0, P.far_a.size() * per_pair * sizeof(double), up_stream_ ? up_stream_ : stream_));
    }
  }
  d_dof_start_ = upload(Lp.dof_start);
  d_dof_inc_ = upload(Lp.dof_inc);
  d_tl_ = upload(P.tl);
  d_tr_ = upload(P.tr);
  as_.node_patch = upload(P.node_patch);
  as_.node_level = upload(P.node_level);
  as_.node_sx = upload(P.node_sx);
  as_.node_sy = upload(P.node_sy);
  for (int c = 1; c <= 3; ++c) {
    as_.sing[c][2] = upload(Lp.sing[c].slot_ab);
    as_.sing[c][3] = upload(Lp.sing[c].slot_ba);
  }
  as_.reg = upload(Lp.reg_ab);
  as_.reg_ba = upload(Lp.reg_ba);
  const long long nnear = static_cast<long long>(Lp.near_row.size());
  const long long nfarp = static_cast<long long>(P.far_a.size());
  d_near_ = dalloc<double>(static_cast<size_t>(nnear) * NL * NL * sw);
  if (stored_couplings()) d_far_ = dalloc<double>(static_cast<size_t>(nfarp) * mm * mm * sw);
  d_img_ = dalloc<double>(static_cast<size_t>(P.n_nodes) * mm * 3);
  bytes_.near = static_cast<size_t>(nnear) * NL * NL * 8 * sw;
  bytes_.far = stored_couplings() ? static_cast<size_t>(nfarp) * mm * mm * 8 * sw : 0;
}

static GeoArgs geo_args(const Discretization& d, const double* cells, const int* el_cell, const double* tab_a,
                        const double* tab_b, const double* kp4) {
  GeoArgs g;
  g.cells = cells;
  g.el_cell = el_cell;
  g.tab_a = tab_a;
  g.tab_b = tab_b;
  g.level = d.level();
  g.epp = d.elements_per_patch();
  g.h = 1.0 / (1 << d.level());
  g.kp.kr = kp4[0];
  g.kp.ki = kp4[1];
  g.kp.dwx = kp4[2];
  g.kp.dwy = kp4[3];
  return g;
}

// K1 element caches + moments, K5 singular integrals (compact blocks)
template <class KT>
void H2Device::launch_element_phase(cudaEvent_t* ev, int& launched) {
  constexpr int NL = KT::NL, NC = KT::NC;
  const Discretization& d = *disc_;
  const int ne = d.element_count(), m = opt_.m, nf = nfar_, nq = nf * nf;
  const GeoArgs g = geo_args(d, d_cells_, d_el_cell_, d_tab_a_, d_tab_b_, as_.kp);
  {
    const size_t smem = (104 + KT::TABN + static_cast<size_t>(nq) * NC * NL) * 8;
    IGB_CUDA(cudaFuncSetAttribute(k_element<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (ne > 0) {
      k_element<KT><<<ne, 128, smem, stream_>>>(g, nf, as_.gxf, as_.gwf, m, as_.lag, d_cpts_, d_cval_, d_mom_);
      ++launched;
    }
    IGB_CUDA(cudaGetLastError());
  }
  IGB_CUDA(cudaEventRecord(ev[kEvElements], stream_));
  auto launch = [&](auto cls_tag, int evi) {
    constexpr int CLS = decltype(cls_tag)::value;
    const SingList& L = sing_items_[CLS];
    if (!L.ea.empty()) {
      SingArgs A;
      A.n_pairs = static_cast<int>(L.ea.size());
      A.n = nsing_;
      A.ea = as_.sing[CLS][0];
      A.eb = as_.sing[CLS][1];
      A.map_a = as_.singm[CLS][0];
      A.map_b = as_.singm[CLS][1];
      A.gx = as_.gxs;
      A.gw = as_.gws;
      A.out = d_sing_blk_[CLS];
      launch_singular<KT, CLS>(g, A, stream_);
      ++launched;
      IGB_CUDA(cudaGetLastError());
    }
    IGB_CUDA(cudaEventRecord(ev[evi], stream_));
  };
  launch(std::integral_constant<int, 3>{}, kEvCoincident);
  launch(std::integral_constant<int, 2>{}, kEvEdge);
  launch(std::integral_constant<int, 1>{}, kEvVertex);
}

// K2 images, K3 couplings (stored mode), K4 regular near, singular scatter
template <class KT>
void H2Device::launch_plan_phase(cudaEvent_t* ev, int& launched) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NC = KT::NC;
  const Discretization& d = *disc_;
  const H2Plan& P = plan_;
  const int m = P.m, mm = m * m, nq = P.nfar * P.nfar;
  const int sw = sizeof(S) / 8;
  const long long nfarp = static_cast<long long>(P.far_a.size());
  const GeoArgs g = geo_args(d, d_cells_, d_el_cell_, d_tab_a_, d_tab_b_, as_.kp);
  {
    const long long tot = static_cast<long long>(P.n_nodes) * mm;
    PatchDev pd{d_patch_info_, d_knots_};
    k_images<<<grid_for(tot, 256), 256, 0, stream_>>>(P.n_nodes, m, as_.cheb, as_.node_patch, as_.node_level,
                                                       as_.node_sx, as_.node_sy, pd, d_cells_, d_img_);
    ++launched;
    IGB_CUDA(cudaGetLastError());
  }
  IGB_CUDA(cudaEventRecord(ev[kEvImages], stream_));
  if (nfarp > 0 && stored_couplings()) {  // fused mode evaluates the couplings inside the matvec
    k_couplings<KT><<<148 * 16, 256, 0, stream_>>>(nfarp, mm, d_far_a_, d_far_b_, d_img_, g.kp, d_far_);
    ++launched;
    IGB_CUDA(cudaGetLastError());
  }
  IGB_CUDA(cudaEventRecord(ev[kEvCouplings], stream_));
  if (!lp_.reg_ab.empty()) {
    const int npair = static_cast<int>(lp_.reg_ab.size());
    const int per = std::max(1, 128 / (NC * nq));  // pairs per CTA: one work item per thread
    const size_t smem = static_cast<size_t>(per) * NC * nq * NL * 8 * sw;
    IGB_CUDA(cudaFuncSetAttribute(k_regular<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (smem > 200 * 1024) throw std::invalid_argument("B200 H2: far quadrature order too large");
    k_regular<KT><<<static_cast<unsigned>((npair + per - 1) / per), 128, smem, stream_>>>(
        npair, per, as_.reg, as_.reg_ba, d_near_a_, d_near_b_, d_near_rs_, d_near_ea_, nq, d_cpts_, d_cval_, g.kp,
        d_near_);
    ++launched;
    IGB_CUDA(cudaGetLastError());
  }
  IGB_CUDA(cudaEventRecord(ev[kEvRegular], stream_));
  for (int c = 3; c >= 1; --c) {
    const size_t n = lp_.sing[c].ea.size();
    if (n == 0) continue;
    k_sing_scatter<S, NL><<<static_cast<unsigned>(n), 128, 0, stream_>>>(
        as_.sing[c][2], as_.sing[c][3], d_near_a_, d_near_rs_, reinterpret_cast<const S*>(d_sing_blk_[c]),
        reinterpret_cast<S*>(d_near_));
    ++launched;
    IGB_CUDA(cudaGetLastError());
  }
  IGB_CUDA(cudaEventRecord(ev[kEvScatter], stream_));
}

void H2Device::collect_times(cudaEvent_t* ev) {
  float ms = 0;
  auto el = [&](int a, int b) {
    IGB_CUDA(cudaEventElapsedTime(&ms, ev[a], ev[b]));
    return static_cast<double>(ms);
  };
  times_.elements = el(kEvStart, kEvElements);
  times_.singular[3] = el(kEvElements, kEvCoincident);
  times_.singular[2] = el(kEvCoincident, kEvEdge);
  times_.singular[1] = el(kEvEdge, kEvVertex);
  times_.images = el(kEvPlanPhase, kEvImages);
  times_.couplings = el(kEvImages, kEvCouplings);
  times_.regular = el(kEvCouplings, kEvRegular);
  times_.scatter = el(kEvRegular, kEvScatter);
  // kernel time (the construction-time gap waiting for the host partition excluded)
  times_.total_device = el(kEvStart, kEvVertex) + el(kEvPlanPhase, kEvScatter);
}

template <class KT>
void H2Device::run_assembly() {
  cudaEvent_t ev[kAsmEvents];
  for (auto& e : ev) IGB_CUDA(cudaEventCreate(&e));
  int launched = 0;
  IGB_CUDA(cudaEventRecord(ev[kEvStart], stream_));
  launch_element_phase<KT>(ev, launched);
  IGB_CUDA(cudaEventRecord(ev[kEvUploaded], stream_));
  IGB_CUDA(cudaEventRecord(ev[kEvPlanPhase], stream_));
  launch_plan_phase<KT>(ev, launched);
  IGB_CUDA(cudaStreamSynchronize(stream_));
  collect_times(ev);
  for (auto& e : ev) cudaEventDestroy(e);
  ++assembly_launches_count_;
  assembly_kernels_ = launched;
}

double H2Device::reassemble() {
  IGB_CUDA(cudaSetDevice(device_));
  // the assembly rewrites the operator arrays: matvecs queued on any stream
  // (apply_device on a caller's stream, DistH2Matrix phases) must finish first
  IGB_CUDA(cudaDeviceSynchronize());
  dispatch_kind([&](auto kt) { run_assembly<decltype(kt)>(); });
  return times_.total_device;
}

// Matvec, phase 1 (h2.cpp:271-310): coefficient gather, near rows on the
// forked side stream, leaf moments and upward transfer of the owned clusters,
// and (multi-GPU) the all-gather payload.
template <class KT>
void H2Device::enqueue_phase1(const double* xin, double* send, cudaStream_t s, cudaEvent_t* pev, int& launches) {
  using S = typename KT::S;
  constexpr int NL = KT::NL;
  const Discretization& d = *disc_;
  const H2Plan& P = plan_;
  const LocalPlan& Lp = lp_;
  const int ne = d.element_count(), m = P.m, mm = m * m, rows = nch_ * mm, L = P.depth;
  const int np = P.n_patches, npp = P.npp, epp = d.elements_per_patch();
  const int nel = static_cast<int>(Lp.el.size());
  const S* x = reinterpret_cast<const S*>(xin);
  S* coef = reinterpret_cast<S*>(d_coef_);
  S* up = reinterpret_cast<S*>(d_up_);
  auto mark = [&](int i) {
    if (pev) IGB_CUDA(cudaEventRecord(pev[i], s));
  };
  mark(0);
  const int nloc = ne * NL;
  pdl_launch(k_coef<S>, grid_for(nloc, 256), 256, 0, s, nloc, x, d_l2g_, d_lsign_, coef);
  ++launches;
  mark(1);
  // near-field rows (HBM-bound) run on a forked stream, overlapping the
  // latency-bound upward/downward passes and the FP64-bound far field
  S* nrows = reinterpret_cast<S*>(d_nrows_);
  if (pev == nullptr && !near_in_phase2_) {
    IGB_CUDA(cudaEventRecord(ev_fork_, s));
    IGB_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    k_near_rows<S, NL><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, side_>>>(
        nel, d_near_rs_, d_near_b_, reinterpret_cast<const S*>(d_near_), coef, nrows);
    ++launches;
    IGB_CUDA(cudaEventRecord(ev_join_, side_));
  }
  pdl_launch(k_leaf_up<S, NL>, grid_for(static_cast<long long>(nel) * rows, 256), 256, 0, s, 
      nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, coef, up);
  ++launches;
  mark(2);
  for (int l = L - 1; l >= 1; --l) {
    const long long tot = static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * (l - 1))) * rows;
    launch_up_level<S>(grid_for(tot, 256), s, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                       d_tl_, d_tr_, up, Lp.c0, Lp.c1);
    ++launches;
  }
  if (Lp.world > 1 && Lp.pack_nodes.size()) {
    const long long tot = static_cast<long long>(Lp.pack_nodes.size()) * rows;
    pdl_launch(k_pack<S>, grid_for(tot, 256), 256, 0, s, static_cast<int>(Lp.pack_nodes.size()), d_pack_nodes_, rows, up,
                                                  reinterpret_cast<S*>(send ? send : d_send_));
    ++launches;
  }
}

// Matvec, phase 2 (h2.cpp:291-376): (multi-GPU) unpack the gathered moments,
// root transfer, far field of the owned targets, downward transfer, leaf
// backward transform + near rows, deterministic DOF gather.
template <class KT>
void H2Device::enqueue_phase2(const double* recv, double* yout, cudaStream_t s, cudaEvent_t* pev, int& launches) {
  using S = typename KT::S;
  constexpr int NL = KT::NL;
  const Discretization& d = *disc_;
  const H2Plan& P = plan_;
  const LocalPlan& Lp = lp_;
  const int m = P.m, mm = m * m, rows = nch_ * mm, L = P.depth;
  const int np = P.n_patches, npp = P.npp, epp = d.elements_per_patch();
  const int nel = static_cast<int>(Lp.el.size());
  S* y = reinterpret_cast<S*>(yout);
  S* coef = reinterpret_cast<S*>(d_coef_);
  S* up = reinterpret_cast<S*>(d_up_);
  S* down = reinterpret_cast<S*>(d_down_);
  S* loc = reinterpret_cast<S*>(d_loc_);
  S* nrows = reinterpret_cast<S*>(d_nrows_);
  auto mark = [&](int i) {
    if (pev) IGB_CUDA(cudaEventRecord(pev[i], s));
  };
  if (pev == nullptr && near_in_phase2_) {  // graph mode: near rows overlap all of phase 2
    IGB_CUDA(cudaEventRecord(ev_fork_, s));
    IGB_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    k_near_rows<S, NL><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, side_>>>(
        nel, d_near_rs_, d_near_b_, reinterpret_cast<const S*>(d_near_), coef, nrows);
    ++launches;
    IGB_CUDA(cudaEventRecord(ev_join_, side_));
  }
  if (Lp.world > 1) {
    const long long tot = static_cast<long long>(Lp.world) * Lp.pack_max * rows;
    pdl_launch(k_unpack<S>, grid_for(tot, 256), 256, 0, s, Lp.world * Lp.pack_max, d_unpack_nodes_, rows,
                                                    reinterpret_cast<const S*>(recv ? recv : d_recv_), up);
    ++launches;
  }
  if (L >= 1) {  // roots (replicated on every rank)
    const long long tot = static_cast<long long>(np) * rows;
    launch_up_level<S>(grid_for(tot, 256), s, np, 0, npp, P.level_offset[0], P.level_offset[1], m, nch_, d_tl_,
                       d_tr_, up, 0, 0);
    ++launches;
  }
  mark(3);
  const size_t ndown = static_cast<size_t>(P.n_nodes) * rows;
  pdl_launch(k_zero<S>, grid_for(static_cast<long long>(ndown), 256), 256, 0, s, ndown, down);
  ++launches;
  mark(4);
  if (n_far_targets_ > 0) {
    const unsigned grid = grid_for(static_cast<long long>(n_far_targets_) * 32, 256);
    if (stored_couplings()) {
      S dw;
      if constexpr (sizeof(S) == 8) {
        dw = 1.0;
      } else {
        const cplx kap = d.kappa();
        const cplx w = d.is_vector() ? -1.0 / (kap * kap) : cplx(1.0, 0.0);
        dw = mk(w.real(), w.imag());
      }
      const S* K = reinterpret_cast<const S*>(d_far_);
      if (mm >= 32) {  // one CTA per target
        const size_t smem = static_cast<size_t>(8) * nch_ * mm * sizeof(S);
        const unsigned nt = static_cast<unsigned>(n_far_targets_);
        if (nch_ == 4) {
          if (mm <= 32) k_far_cta<S, 4, 1><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else if (mm <= 64) k_far_cta<S, 4, 2><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else k_far_cta<S, 4, 4><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        } else {
          if (mm <= 32) k_far_cta<S, 1, 1><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else if (mm <= 64) k_far_cta<S, 1, 2><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else k_far_cta<S, 1, 4><<<nt, 256, smem, s>>>(d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        }
      } else if (nch_ == 4) {
        if (mm <= 32) k_far<S, 4, 1><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else if (mm <= 64) k_far<S, 4, 2><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else k_far<S, 4, 4><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
      } else {
        if (mm <= 32) k_far<S, 1, 1><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else if (mm <= 64) k_far<S, 1, 2><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else k_far<S, 1, 4><<<grid, 256, 0, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, K, mm, up, dw, down);
      }
    } else if (sym_far_) {
      const unsigned gsym = grid_for(static_cast<long long>(n_sym_targets_) * 32, 256);
      double* dn = reinterpret_cast<double*>(down);
      const double* upd = reinterpret_cast<const double*>(up);
      if (far_col_) {  // one GPU, m <= 5 (graphs without the level split: depth 0)
        switch (m) {
          case 2: k_far_col<2, 4, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          case 3: k_far_col<3, 4, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          case 4: k_far_col<4, 3, 2><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          default: k_far_col<5, 2, 2><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
        }
      } else if (m <= 5) {  // ranks: column stream over the rank's pair lists
#define IGB_FCL(M_, MB_, C_)                                                                                 \
  k_far_col_list<M_, MB_, C_><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_col_rs_, d_col_q_, d_far_b_, \
                                                   d_trans_, d_img_, upd, dn, d_slot_)
        switch (m) {
          case 2: IGB_FCL(2, 4, 1); break;
          case 3: IGB_FCL(3, 4, 1); break;
          case 4: IGB_FCL(4, 3, 2); break;
          default: IGB_FCL(5, 2, 2); break;
        }
#undef IGB_FCL
      } else if (lp_.world > 1) {  // m = 6: the lane-tile kernel (one-sided pairs with other ranks' nodes)
        k_far_sym<6, true, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_,
                                                   d_far_b_, d_trans_, d_img_, upd, dn, d_slot_, d_owned_, 1);
      } else {
        k_far_sym<6, false, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_,
                                                    d_far_b_, d_trans_, d_img_, upd, dn, d_slot_, d_owned_, 0);
      }
      ++launches;
      if (lp_.world > 1)
        pdl_launch(k_far_lower<true>, grid_for(static_cast<long long>(P.n_nodes) * mm, 256), 256, 0, s, 
            P.n_nodes, mm, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, dn, 0, 1, 0);
      else
        pdl_launch(k_far_lower<false>, grid_for(static_cast<long long>(P.n_nodes) * mm, 256), 256, 0, s, 
            P.n_nodes, mm, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, dn, 0, 1, 0);
    } else if (sym_w_) {
      KParams kp;
      kp.kr = as_.kp[0];
      kp.ki = as_.kp[1];
      kp.dwx = as_.kp[2];
      kp.dwy = as_.kp[3];
      constexpr int PW = ((4 + KT::NC * static_cast<int>(sizeof(S) / 8)) + 1) / 2 * 2;
      const unsigned gsym = grid_for(static_cast<long long>(n_sym_targets_) * 32, 256);
      S* sl = reinterpret_cast<S*>(d_slot_);
      const int R = (mm + 31) / 32;
      const size_t smem = static_cast<size_t>(8) * 32 * R * PW * 8;
      if (R == 1)
        k_far_sym_w<KT, 1><<<gsym, 256, smem, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else if (R == 2)
        k_far_sym_w<KT, 2><<<gsym, 256, smem, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else if (R == 3)
        k_far_sym_w<KT, 3><<<gsym, 256, smem, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else
        k_far_sym_w<KT, 4><<<gsym, 256, smem, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      ++launches;
      const int stride = rows * static_cast<int>(sizeof(S) / 8);
      pdl_launch(k_far_lower<false>, grid_for(static_cast<long long>(P.n_nodes) * stride, 256), 256, 0, s, 
          P.n_nodes, stride, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, reinterpret_cast<double*>(down), 0, 1, 0);
    } else {
      KParams kp;
      kp.kr = as_.kp[0];
      kp.ki = as_.kp[1];
      kp.dwx = as_.kp[2];
      kp.dwy = as_.kp[3];
      constexpr int PW = ((4 + KT::NC * static_cast<int>(sizeof(S) / 8)) + 1) / 2 * 2;
      if (mm <= 32) {
        const size_t smem = 8 * 32 * 1 * PW * 8;
        k_far_fused<KT, 1><<<grid, 256, smem, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, d_img_, mm, up, kp, down);
      } else if (mm <= 64) {
        const size_t smem = 8 * 32 * 2 * PW * 8;
        k_far_fused<KT, 2><<<grid, 256, smem, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, d_img_, mm, up, kp, down);
      } else {
        const size_t smem = 8 * 32 * 4 * PW * 8;
        k_far_fused<KT, 4><<<grid, 256, smem, s>>>(n_far_targets_, d_far_targets_, d_far_rs_, d_far_b_, d_img_, mm, up, kp, down);
      }
    }
    ++launches;
  }
  mark(5);
  if (far_only_) {  // introspection: stop after the far field (phase 4)
    if (pev == nullptr) IGB_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    return;
  }
  if (pev != nullptr) {  // profiling: the near rows serialised as their own phase
    k_near_rows<S, NL><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, s>>>(
        nel, d_near_rs_, d_near_b_, reinterpret_cast<const S*>(d_near_), coef, nrows);
    ++launches;
  }
  mark(6);
  for (int l = 0; l < L; ++l) {
    const long long tot = static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * l)) * rows;
    launch_down_level<S>(grid_for(tot, 256), s, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                         d_tl_, d_tr_, down, Lp.c0, Lp.c1);
    ++launches;
  }
  if (pev == nullptr) IGB_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));  // near rows (side stream) done
  pdl_launch(k_leaf_down<S, NL>, grid_for(static_cast<long long>(nel) * NL, 256), 256, 0, s, 
      nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, down, nrows, loc);
  ++launches;
  mark(7);
  pdl_launch(k_scatter<S>, grid_for(d.dof_count(), 256), 256, 0, s, d.dof_count(), d_dof_start_, d_dof_inc_, d_loc_sign_, loc, y);
  ++launches;
  mark(8);
  IGB_CUDA(cudaGetLastError());
}

template <class KT>
void H2Device::enqueue_apply(const double* xin, double* yout, cudaStream_t s, cudaEvent_t* pev) {
  int launches = 0;
  enqueue_phase1<KT>(xin, nullptr, s, pev, launches);
  enqueue_phase2<KT>(nullptr, yout, s, pev, launches);
  apply_launches_ = launches;
}

// Single-GPU matvec graph split by tree level (symmetric far field).  Far pairs
// join clusters of one level, and most of them sit on the leaf level, which
// only needs the leaf moments.  Main stream: coefficients, leaf moments, zero,
// leaf-level far field + its transposed slots, last downward level, leaf
// transform, gather.  Side stream 2, concurrently: upward pass, coarse-level
// far field + slots, downward levels above the leaves.  Side stream 1: near rows.
template <class KT>
void H2Device::enqueue_apply_split(const double* xin, double* yout, cudaStream_t s, KernelMarks* prof) {
  using S = typename KT::S;
  constexpr int NL = KT::NL;
  const Discretization& d = *disc_;
  const H2Plan& P = plan_;
  const LocalPlan& Lp = lp_;
  const int m = P.m, mm = m * m, rows = nch_ * mm, L = P.depth;
  const int np = P.n_patches, npp = P.npp, epp = d.elements_per_patch();
  const int nel = static_cast<int>(Lp.el.size()), nloc = d.element_count() * NL;
  const S* x = reinterpret_cast<const S*>(xin);
  S* y = reinterpret_cast<S*>(yout);
  S* coef = reinterpret_cast<S*>(d_coef_);
  S* up = reinterpret_cast<S*>(d_up_);
  S* down = reinterpret_cast<S*>(d_down_);
  S* loc = reinterpret_cast<S*>(d_loc_);
  S* nrows = reinterpret_cast<S*>(d_nrows_);
  double* dn = reinterpret_cast<double*>(down);
  const double* upd = reinterpret_cast<const double*>(up);
  int launches = 0;
  (void)nloc;
  (void)coef;
  const bool fused = KT::KIND == 0 && NL <= 16 && n_near_rest_ >= 0;
  // profiling (prof != nullptr): the same kernels serialised on s, an event
  // after each one, so every graph kernel is timed on its own
  cudaStream_t side1 = prof ? s : side_, side2 = prof ? s : side2_;
  auto tick = [&](const char* name) {
    if (!prof) return;
    cudaEvent_t e;
    IGB_CUDA(cudaEventCreate(&e));
    IGB_CUDA(cudaEventRecord(e, s));
    prof->emplace_back(name, e);
  };
  tick("start");
  if (!prof) {
    IGB_CUDA(cudaEventRecord(ev_fork_, s));
    IGB_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
  }
  if (!fused) {
    k_near_rows<S, NL, true><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, side1>>>(
        nel, d_near_rs_, d_near_b_, reinterpret_cast<const S*>(d_near_), x, nrows, d_l2g_, d_lsign_);
    ++launches;
    tick("near_rows");
  }
  if (!prof) IGB_CUDA(cudaEventRecord(ev_join_, side_));
  const long long ndown = static_cast<long long>(P.n_nodes) * rows;
  pdl_launch(k_leaf_up_x<S, NL>, grid_for(std::max(ndown, static_cast<long long>(nel) * rows), 256), 256, 0, s, 
      nel, rows, epp, npp, P.level_offset[L], d_mom_, x, d_l2g_, d_lsign_, up, down, ndown);
  ++launches;
  tick("leaf_up");
  if (!prof) {
    IGB_CUDA(cudaEventRecord(ev_fork2_, s));
    IGB_CUDA(cudaStreamWaitEvent(side2_, ev_fork2_, 0));
  }
  auto far_sym = [&](cudaStream_t st, int n, const int* targets) {
    if (n == 0) return;
    const unsigned g = grid_for(static_cast<long long>(n) * 32, 256);
    if (far_col_) {  // column stream: m <= 5
#define IGB_FC(M_, MB_, C_) k_far_col<M_, MB_, C_><<<g, 256, 0, st>>>(n, targets, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_)
      switch (m) {
        case 2: IGB_FC(2, 4, 1); break;
        case 3: IGB_FC(3, 4, 1); break;
        case 4: IGB_FC(4, 3, 2); break;
        default: IGB_FC(5, 2, 2); break;
      }
#undef IGB_FC
      ++launches;
      return;
    }
    k_far_sym<6, false, 1><<<g, 256, 0, st>>>(n, targets, d_upper_start_, d_far_rs_, d_far_b_, d_trans_, d_img_,
                                              upd, dn, d_slot_, d_owned_, 0);  // m = 6: lane tile
    ++launches;
  };
  auto far_lower = [&](cudaStream_t st, int which) {
    pdl_launch(k_far_lower<false>, grid_for(static_cast<long long>(P.n_nodes) * mm, 256), 256, 0, st, 
        P.n_nodes, mm, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, dn, which, npp, P.level_offset[L]);
    ++launches;
  };
  // side stream 2: upward pass, coarse far field, downward levels 0 .. L-2
  for (int l = L - 1; l >= 0; --l) {
    const long long tot = (l == 0 ? static_cast<long long>(np) : static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * (l - 1)))) * rows;
    launch_up_level<S>(grid_for(tot, 256), side2, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                       d_tl_, d_tr_, up, l == 0 ? 0 : Lp.c0, l == 0 ? 0 : Lp.c1);
    ++launches;
  }
  tick("upward");
  far_sym(side2, n_sym_coarse_, d_sym_coarse_);
  tick("far_coarse");
  far_lower(side2, 2);
  tick("far_lower_coarse");
  for (int l = 0; l + 1 < L && !far_only_; ++l) {
    const long long tot = static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * l)) * rows;
    launch_down_level<S>(grid_for(tot, 256), side2, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                         d_tl_, d_tr_, down, Lp.c0, Lp.c1);
    ++launches;
  }
  tick("downward_coarse");
  if (!prof) IGB_CUDA(cudaEventRecord(ev_join2_, side2_));
  // main: leaf-level far field (fused with the near rows when enabled)
  if (fused) {
    if constexpr (KT::KIND == 0 && NL <= 16) {
      const long long nw = static_cast<long long>(n_sym_fine_) + n_near_rest_;
      auto fused_launch = [&](auto kern) {
        kern<<<grid_for(nw * 32, 256), 256, 0, s>>>(
            n_sym_fine_, d_sym_fine_, n_near_rest_, d_near_rest_, epp, npp, P.level_offset[L], d_upper_start_,
            d_far_rs_, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_, d_owned_, d_near_rs_, d_near_b_,
            reinterpret_cast<const double*>(d_near_), reinterpret_cast<const double*>(x),
            reinterpret_cast<double*>(nrows), d_l2g_, d_lsign_);
      };
      if (m == 4)
        fused_launch(k_far_col_near<4, NL, 3, 2>);
      else
        fused_launch(k_far_col_near<5, NL, 2, 2>);
      ++launches;
    }
  } else {
    far_sym(s, n_sym_fine_, d_sym_fine_);
  }
  tick(fused ? "far_leaf_near" : "far_leaf");
  far_lower(s, 1);
  tick("far_lower_leaf");
  if (!prof) IGB_CUDA(cudaStreamWaitEvent(s, ev_join2_, 0));
  if (far_only_) {  // introspection: stop after the far field (phase 4)
    if (!prof) IGB_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
    return;
  }
  {
    const int l = L - 1;
    const long long tot = static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * l)) * rows;
    launch_down_level<S>(grid_for(tot, 256), s, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                         d_tl_, d_tr_, down, Lp.c0, Lp.c1);
    ++launches;
  }
  tick("downward_leaf");
  if (!prof) IGB_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
  pdl_launch(k_leaf_down<S, NL>, grid_for(static_cast<long long>(nel) * NL, 256), 256, 0, s, 
      nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, down, nrows, loc);
  tick("leaf_down");
  pdl_launch(k_scatter<S>, grid_for(d.dof_count(), 256), 256, 0, s, d.dof_count(), d_dof_start_, d_dof_inc_, d_loc_sign_, loc, y);
  launches += 2;
  tick("scatter");
  IGB_CUDA(cudaGetLastError());
  apply_launches_ = launches;
}

template <class F>
void H2Device::dispatch_kind(F&& f) {
  const int kind = disc_->kind();
  const int q = kind == kMaxwell ? disc_->degree() : disc_->scalar_degree();
  if (kind == kLaplace) {
    switch (q) {
      case 0: f(LapT<0>{}); break;
      case 1: f(LapT<1>{}); break;
      case 2: f(LapT<2>{}); break;
      case 3: f(LapT<3>{}); break;
      default: f(LapT<4>{}); break;
    }
  } else if (kind == kHelmholtz) {
    switch (q) {
      case 0: f(HelmT<0>{}); break;
      case 1: f(HelmT<1>{}); break;
      case 2: f(HelmT<2>{}); break;
      case 3: f(HelmT<3>{}); break;
      default: f(HelmT<4>{}); break;
    }
  } else {
    switch (q) {
      case 1: f(MaxT<1>{}); break;
      case 2: f(MaxT<2>{}); break;
      default: f(MaxT<3>{}); break;
    }
  }
}

// Multi-GPU matvec phases as two CUDA graphs over the handle's buffers (one
// graph launch each instead of ~20 kernel launches); the caller's collectives
// run between them on its stream.  The near rows are forked at the start of
// phase 2 (coefficients come from phase 1) and joined before the leaf transform.
void H2Device::dist_phase1(const double* x, double* send, cudaStream_t s) {
  IGB_CUDA(cudaSetDevice(device_));
  const size_t sw = is_complex() ? 16 : 8;
  if (!graph1_) {
    cudaGraph_t graph;
    int n = 0;
    near_in_phase2_ = true;
    IGB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    dispatch_kind([&](auto kt) { enqueue_phase1<decltype(kt)>(dx_, d_send_, stream_, nullptr, n); });
    IGB_CUDA(cudaStreamEndCapture(stream_, &graph));
    IGB_CUDA(cudaGraphInstantiate(&graph1_, graph, 0));
    cudaGraphDestroy(graph);
    phase1_launches_ = n;
  }
  IGB_CUDA(cudaMemcpyAsync(dx_, x, static_cast<size_t>(dim()) * sw, cudaMemcpyDeviceToDevice, s));
  IGB_CUDA(cudaGraphLaunch(graph1_, s));
  if (lp_.world > 1 && send_count() > 0 && send != nullptr)  // one rank: nothing is exchanged
    IGB_CUDA(cudaMemcpyAsync(send, d_send_, send_count() * sw, cudaMemcpyDeviceToDevice, s));
}
void H2Device::dist_phase2(const double* recv, double* y, cudaStream_t s) {
  IGB_CUDA(cudaSetDevice(device_));
  const size_t sw = is_complex() ? 16 : 8;
  if (!graph2_) {
    cudaGraph_t graph;
    int n = 0;
    near_in_phase2_ = true;
    IGB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    dispatch_kind([&](auto kt) { enqueue_phase2<decltype(kt)>(d_recv_, dy_, stream_, nullptr, n); });
    IGB_CUDA(cudaStreamEndCapture(stream_, &graph));
    IGB_CUDA(cudaGraphInstantiate(&graph2_, graph, 0));
    cudaGraphDestroy(graph);
    apply_launches_ = phase1_launches_ + n;
  }
  if (lp_.world > 1 && send_count() > 0)
    IGB_CUDA(cudaMemcpyAsync(d_recv_, recv, send_count() * lp_.world * sw, cudaMemcpyDeviceToDevice, s));
  IGB_CUDA(cudaGraphLaunch(graph2_, s));
  IGB_CUDA(cudaMemcpyAsync(y, dy_, static_cast<size_t>(dim()) * sw, cudaMemcpyDeviceToDevice, s));
}

void H2Device::enqueue_apply_dispatch(const double* x, double* y, cudaStream_t s, cudaEvent_t* pev) {
  const int kind = disc_->kind();
  const int q = kind == kMaxwell ? disc_->degree() : disc_->scalar_degree();
  if (kind == kLaplace) {
    switch (q) {
      case 0: enqueue_apply<LapT<0>>(x, y, s, pev); break;
      case 1: enqueue_apply<LapT<1>>(x, y, s, pev); break;
      case 2: enqueue_apply<LapT<2>>(x, y, s, pev); break;
      case 3: enqueue_apply<LapT<3>>(x, y, s, pev); break;
      default: enqueue_apply<LapT<4>>(x, y, s, pev); break;
    }
  } else if (kind == kHelmholtz) {
    switch (q) {
      case 0: enqueue_apply<HelmT<0>>(x, y, s, pev); break;
      case 1: enqueue_apply<HelmT<1>>(x, y, s, pev); break;
      case 2: enqueue_apply<HelmT<2>>(x, y, s, pev); break;
      case 3: enqueue_apply<HelmT<3>>(x, y, s, pev); break;
      default: enqueue_apply<HelmT<4>>(x, y, s, pev); break;
    }
  } else {
    switch (q) {
      case 1: enqueue_apply<MaxT<1>>(x, y, s, pev); break;
      case 2: enqueue_apply<MaxT<2>>(x, y, s, pev); break;
      default: enqueue_apply<MaxT<3>>(x, y, s, pev); break;
    }
  }
}

void H2Device::launch_apply_graph(cudaStream_t s) {
  if (lp_.world > 1)
    throw std::logic_error(
        "H2Matrix: a rank of a distributed operator is applied with dist_phase1 / all-gather / dist_phase2 / "
        "all-reduce (DistH2Matrix)");
  IGB_CUDA(cudaSetDevice(device_));
  if (!graph_exec_) {
    cudaGraph_t graph;
    IGB_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    if (split_graph())
      dispatch_kind([&](auto kt) {
        if constexpr (decltype(kt)::KIND == 0) enqueue_apply_split<decltype(kt)>(dx_, dy_, stream_);
      });
    else
      enqueue_apply_dispatch(dx_, dy_, stream_, nullptr);
    IGB_CUDA(cudaStreamEndCapture(stream_, &graph));
    IGB_CUDA(cudaGraphInstantiate(&graph_exec_, graph, 0));
    cudaGraphDestroy(graph);
  }
  IGB_CUDA(cudaGraphLaunch(graph_exec_, s));
}

void H2Device::profile_apply(int iters, double* phase_ms) {
  IGB_CUDA(cudaSetDevice(device_));
  cudaEvent_t ev[9];
  for (auto& e : ev) IGB_CUDA(cudaEventCreate(&e));
  for (int k = 0; k < 8; ++k) phase_ms[k] = 0.0;
  for (int it = 0; it < iters; ++it) {
    enqueue_apply_dispatch(dx_, dy_, stream_, ev);
    IGB_CUDA(cudaStreamSynchronize(stream_));
    for (int k = 0; k < 8; ++k) {
      float ms = 0;
      IGB_CUDA(cudaEventElapsedTime(&ms, ev[k], ev[k + 1]));
      phase_ms[k] += ms;
    }
  }
  for (auto& e : ev) cudaEventDestroy(e);
}

void H2Device::far_field(const double* x, double* up_out, double* down_out) {
  if (lp_.world > 1) throw std::logic_error("far_field: not available on a rank of a distributed operator");
  IGB_CUDA(cudaSetDevice(device_));
  const size_t sw = is_complex() ? 16 : 8;
  IGB_CUDA(cudaDeviceSynchronize());
  IGB_CUDA(cudaMemcpy(dx_, x, static_cast<size_t>(dim()) * sw, cudaMemcpyHostToDevice));
  far_only_ = true;
  try {
    if (split_graph())
      dispatch_kind([&](auto kt) {
        if constexpr (decltype(kt)::KIND == 0) enqueue_apply_split<decltype(kt)>(dx_, dy_, stream_);
      });
    else
      enqueue_apply_dispatch(dx_, dy_, stream_, nullptr);
  } catch (...) {
    far_only_ = false;
    throw;
  }
  far_only_ = false;
  IGB_CUDA(cudaStreamSynchronize(stream_));
  const size_t n = static_cast<size_t>(plan_.n_nodes) * nch_ * plan_.m * plan_.m * sw;
  if (up_out) IGB_CUDA(cudaMemcpy(up_out, d_up_, n, cudaMemcpyDeviceToHost));
  if (down_out) IGB_CUDA(cudaMemcpy(down_out, d_down_, n, cudaMemcpyDeviceToHost));
}

std::vector<std::pair<std::string, double>> H2Device::profile_kernels(int iters) {
  IGB_CUDA(cudaSetDevice(device_));
  if (!split_graph()) throw std::logic_error("profile_kernels: only the single-GPU level-split graph");
  std::vector<std::pair<std::string, double>> out;
  for (int it = 0; it < iters; ++it) {
    KernelMarks marks;
    dispatch_kind([&](auto kt) {
      if constexpr (decltype(kt)::KIND == 0) enqueue_apply_split<decltype(kt)>(dx_, dy_, stream_, &marks);
    });
    IGB_CUDA(cudaStreamSynchronize(stream_));
    if (out.empty())
      for (size_t k = 1; k < marks.size(); ++k) out.emplace_back(marks[k].first, 0.0);
    for (size_t k = 1; k < marks.size(); ++k) {
      float ms = 0;
      IGB_CUDA(cudaEventElapsedTime(&ms, marks[k - 1].second, marks[k].second));
      out[k - 1].second += ms;
    }
    for (auto& mk : marks) cudaEventDestroy(mk.second);
  }
  return out;
}

double H2Device::bench_steps(int steps, int matvecs, double* assembly_ms) {
  IGB_CUDA(cudaSetDevice(device_));
  launch_apply_graph(stream_);  // instantiate outside the timed region
  IGB_CUDA(cudaStreamSynchronize(stream_));
  cudaEvent_t a, b;
  IGB_CUDA(cudaEventCreate(&a));
  IGB_CUDA(cudaEventCreate(&b));
  double asm_ms = 0;
  IGB_CUDA(cudaEventRecord(a, stream_));
  for (int st = 0; st < steps; ++st) {
    asm_ms += reassemble();
    for (int i = 0; i < matvecs; ++i) launch_apply_graph(stream_);
  }
  IGB_CUDA(cudaEventRecord(b, stream_));
  IGB_CUDA(cudaEventSynchronize(b));
  float ms = 0;
  IGB_CUDA(cudaEventElapsedTime(&ms, a, b));
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  if (assembly_ms) *assembly_ms = asm_ms;
  return ms;
}

void H2Device::apply_device(const double* x, double* y, cudaStream_t s) {
  const size_t bytes = static_cast<size_t>(dim()) * (is_complex() ? 16 : 8);
  IGB_CUDA(cudaSetDevice(device_));
  if (s == nullptr) s = stream_;
  // dx_ / dy_ are shared by every apply on this handle: order this call after
  // the previous one, whichever stream that ran on
  IGB_CUDA(cudaStreamWaitEvent(s, ev_apply_done_, 0));
  IGB_CUDA(cudaMemcpyAsync(dx_, x, bytes, cudaMemcpyDeviceToDevice, s));
  launch_apply_graph(s);
  IGB_CUDA(cudaMemcpyAsync(y, dy_, bytes, cudaMemcpyDeviceToDevice, s));
  IGB_CUDA(cudaEventRecord(ev_apply_done_, s));
}

static bool is_pinned(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

void H2Device::apply_host(const double* x, double* y) {
  const size_t bytes = static_cast<size_t>(dim()) * (is_complex() ? 16 : 8);
  IGB_CUDA(cudaSetDevice(device_));
  // page-locked caller buffers are copied directly; pageable ones go through
  // the handle's pinned staging buffers
  const bool px = is_pinned(x), py = is_pinned(y);
  if (!h_x_pinned_ && !(px && py)) {
    h_x_pinned_ = static_cast<double*>(pinned_get(bytes));
    h_y_pinned_ = static_cast<double*>(pinned_get(bytes));
  }
  const double* xs = x;
  if (!px) {
    std::memcpy(h_x_pinned_, x, bytes);
    xs = h_x_pinned_;
  }
  double* ys = py ? y : h_y_pinned_;
  IGB_CUDA(cudaStreamWaitEvent(stream_, ev_apply_done_, 0));  // a device apply on another stream
  IGB_CUDA(cudaMemcpyAsync(dx_, xs, bytes, cudaMemcpyHostToDevice, stream_));
  launch_apply_graph(stream_);
  IGB_CUDA(cudaMemcpyAsync(ys, dy_, bytes, cudaMemcpyDeviceToHost, stream_));
  IGB_CUDA(cudaEventRecord(ev_apply_done_, stream_));
  IGB_CUDA(cudaStreamSynchronize(stream_));
  if (!py) std::memcpy(y, h_y_pinned_, bytes);
}

void H2Device::near_blocks(long long first, long long count, double* out) const {
  if (lp_.world > 1)  // a rank holds only its own block rows, in a rank-local layout
    throw std::logic_error("near_blocks: not available on a rank of a distributed operator");
  const int nl = disc_->local_count(), sw = is_complex() ? 2 : 1;
  if (first < 0 || first + count > static_cast<long long>(plan_.near_a.size()))
    throw std::invalid_argument("near_blocks: range out of bounds");
  IGB_CUDA(cudaSetDevice(device_));
  if (count == 0) return;
  // rows touched by the range
  const int e0 = plan_.near_a[first], e1 = plan_.near_a[first + count - 1];
  const int r0 = plan_.near_row_start[e0], r1 = plan_.near_row_start[e1 + 1];
  std::vector<double> buf(static_cast<size_t>(r1 - r0) * nl * nl * sw);
  IGB_CUDA(cudaMemcpy(buf.data(), d_near_ + static_cast<size_t>(r0) * nl * nl * sw, buf.size() * 8,
                      cudaMemcpyDeviceToHost));
  for (long long q = first; q < first + count; ++q) {
    const int e = plan_.near_a[q], rs = plan_.near_row_start[e], cnt = plan_.near_row_start[e + 1] - rs;
    for (int la = 0; la < nl; ++la)
      for (int lb = 0; lb < nl; ++lb) {
        const size_t src = static_cast<size_t>(rs - r0) * nl * nl + (static_cast<size_t>(la) * cnt + (q - rs)) * nl + lb;
        const size_t dst = (static_cast<size_t>(q - first) * nl + la) * nl + lb;
        for (int c = 0; c < sw; ++c) out[dst * sw + c] = buf[src * sw + c];
      }
  }
}
void H2Device::couplings(long long first, long long count, double* out) const {
  if (lp_.world > 1)
    throw std::logic_error("couplings: not available on a rank of a distributed operator");
  const size_t per = static_cast<size_t>(plan_.m) * plan_.m * plan_.m * plan_.m * (is_complex() ? 2 : 1);
  if (first < 0 || first + count > static_cast<long long>(plan_.far_a.size()))
    throw std::invalid_argument("couplings: range out of bounds");
  IGB_CUDA(cudaSetDevice(device_));
  if (count == 0) return;
  if (d_far_) {
    IGB_CUDA(cudaMemcpy(out, d_far_ + first * per, count * per * 8, cudaMemcpyDeviceToHost));
    return;
  }
  // fused mode: evaluate the requested couplings with the assembly kernel
  // (the pair rows are not resident in this mode: upload the slice)
  double* tmp = nullptr;
  int* rows = nullptr;
  IGB_CUDA(cudaMalloc(&tmp, count * per * 8));
  if (cudaMalloc(&rows, count * sizeof(int)) != cudaSuccess) {
    cudaFree(tmp);
    throw std::runtime_error("couplings: out of device memory");
  }
  const cudaError_t e0 = cudaMemcpy(rows, plan_.far_a.data() + first, count * sizeof(int), cudaMemcpyHostToDevice);
  KParams kp;
  kp.kr = as_.kp[0];
  kp.ki = as_.kp[1];
  kp.dwx = as_.kp[2];
  kp.dwy = as_.kp[3];
  const int mm = plan_.m * plan_.m;
  if (e0 == cudaSuccess) {
    if (is_complex())
      k_couplings<HelmT<0>><<<148 * 16, 256, 0, stream_>>>(count, mm, rows, d_far_b_ + first, d_img_, kp, tmp);
    else
      k_couplings<LapT<0>><<<148 * 16, 256, 0, stream_>>>(count, mm, rows, d_far_b_ + first, d_img_, kp, tmp);
  }
  const cudaError_t e1 = cudaStreamSynchronize(stream_);
  const cudaError_t e2 = cudaMemcpy(out, tmp, count * per * 8, cudaMemcpyDeviceToHost);
  cudaFree(tmp);
  cudaFree(rows);
  IGB_CUDA(e0);
  IGB_CUDA(e1);
  IGB_CUDA(e2);
}
void H2Device::moments(double* out) const {
  IGB_CUDA(cudaSetDevice(device_));
  IGB_CUDA(cudaMemcpy(out, d_mom_, bytes_.moments, cudaMemcpyDeviceToHost));
}
void H2Device::images(double* out) const {
  IGB_CUDA(cudaSetDevice(device_));
  IGB_CUDA(cudaMemcpy(out, d_img_, static_cast<size_t>(plan_.n_nodes) * plan_.m * plan_.m * 3 * 8,
                      cudaMemcpyDeviceToHost));
}

// ====================================================== dense assembly
// Dense Galerkin matrix (assembly.cpp:16-53) on one device, column-major
// nd x nd Scalar in `out` (host).  Test elements are processed in chunks that
// fit a ~1 GB block buffer: all (ea, eb) blocks of the chunk (regular tensor
// Gauss, then the singular items from the mesh topology), the row strips
// gathered per trial DOF, and the strips added to the DOF rows in ascending
// test element -- the reference's summation structure.
template <class KT>
static void dense_impl(const Discretization& d, int far_order, int sing_order, int device, double* out) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NC = KT::NC;
  if (d.local_count() != NL) throw std::logic_error("B200 dense: local count mismatch");
  int nf = 0, ns = 0;
  check_h2_options(d, 2, 1.0, far_order, sing_order, &nf, &ns);
  if (ns > 16) throw std::invalid_argument("B200 dense: singular order > 16 not supported");
  int ndev = 0;
  IGB_CUDA(cudaGetDeviceCount(&ndev));
  if (device < 0 || device >= ndev) throw std::invalid_argument("assemble_dense: CUDA device index out of range");
  IGB_CUDA(cudaSetDevice(device));
  const int ne = d.element_count(), nd = d.dof_count(), nq = nf * nf, m = 2;
  std::vector<void*> mem;
  cudaStream_t st = nullptr;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    IGB_CUDA(cudaMalloc(&p, bytes ? bytes : 8));
    mem.push_back(p);
    return p;
  };
  auto up = [&](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* p = static_cast<T*>(alloc(v.size() * sizeof(T)));
    if (!v.empty()) IGB_CUDA(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  };
  try {
    IGB_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    std::vector<double> cells(d.cells().size() * kCellStride, 0.0);
    for (size_t c = 0; c < d.cells().size(); ++c) {
      const GeomCell& gc = d.cells()[c];
      for (int comp = 0; comp < 4; ++comp)
        for (int j = 0; j <= kMaxGeomDeg; ++j)
          for (int i = 0; i <= kMaxGeomDeg; ++i) cells[c * kCellStride + comp * 25 + j * 5 + i] = gc.coef[comp][j][i];
      cells[c * kCellStride + 100] = gc.u0;
      cells[c * kCellStride + 101] = gc.v0;
    }
    const double* d_cells = up(cells);
    const int* d_el_cell = up(d.element_cell());
    const double* d_tab_a = up(d.is_vector() ? d.tab_p() : d.tab_s());
    const double* d_tab_b = up(d.is_vector() ? d.tab_q() : std::vector<double>(1, 0.0));
    const double* d_lsign = up(d.lsign());
    std::vector<double> gxf, gwf, gxs, gws;
    gauss_rule(nf, gxf, gwf);
    gauss_rule(ns, gxs, gws);
    const double *d_gxf = up(gxf), *d_gwf = up(gwf), *d_gxs = up(gxs), *d_gws = up(gws);
    const std::vector<double> cheb = cheb_nodes(m);
    std::vector<double> lag(static_cast<size_t>(m) * nf), tmp(m);
    for (int a = 0; a < nf; ++a) {
      lagrange_all(cheb, gxf[a], tmp.data());
      for (int i = 0; i < m; ++i) lag[i * nf + a] = tmp[i];
    }
    const double* d_lag = up(lag);
    double kp4[4] = {d.kappa().real(), d.kappa().imag(), 0.0, 0.0};
    if (d.is_vector()) {
      const cplx dw = -1.0 / (d.kappa() * d.kappa());
      kp4[2] = dw.real();
      kp4[3] = dw.imag();
    }
    const GeoArgs g = geo_args(d, d_cells, d_el_cell, d_tab_a, d_tab_b, kp4);
    // element caches (+ moments of a 2-point interpolation, unused)
    double* d_cpts = static_cast<double*>(alloc(static_cast<size_t>(ne) * nq * 3 * 8));
    double* d_cval = static_cast<double*>(alloc(static_cast<size_t>(ne) * NC * nq * NL * 8));
    double* d_mom = static_cast<double*>(alloc(static_cast<size_t>(ne) * NL * (d.is_vector() ? 4 : 1) * m * m * 8));
    {
      const size_t smem = (104 + KT::TABN + static_cast<size_t>(nq) * NC * NL) * 8;
      IGB_CUDA(cudaFuncSetAttribute(k_element<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      if (ne > 0) k_element<KT><<<ne, 128, smem, st>>>(g, nf, d_gxf, d_gwf, m, d_lag, d_cpts, d_cval, d_mom);
      IGB_CUDA(cudaGetLastError());
    }
    // singular items (ea <= eb) from the mesh topology, compact blocks
    SingList items[4];
    d.singular_items(nullptr, items);
    const int *d_ia[4] = {}, *d_ib[4] = {};
    S* d_sblk[4] = {};
    {
      using LY = SingLayout<KT>;
      auto launch = [&](auto cls_tag) {
        constexpr int CLS = decltype(cls_tag)::value;
        const SingList& L = items[CLS];
        d_ia[CLS] = up(L.ea);
        d_ib[CLS] = up(L.eb);
        d_sblk[CLS] = static_cast<S*>(alloc(L.ea.size() * NL * NL * sizeof(S)));
        if (L.ea.empty()) return;
        SingArgs A;
        A.n_pairs = static_cast<int>(L.ea.size());
        A.n = ns;
        A.ea = d_ia[CLS];
        A.eb = d_ib[CLS];
        A.map_a = up(L.map_a);
        A.map_b = up(L.map_b);
        A.gx = d_gxs;
        A.gw = d_gws;
        A.out = reinterpret_cast<double*>(d_sblk[CLS]);
        launch_singular<KT, CLS>(g, A, st);
        IGB_CUDA(cudaGetLastError());
      };
      launch(std::integral_constant<int, 3>{});
      launch(std::integral_constant<int, 2>{});
      launch(std::integral_constant<int, 1>{});
    }
    // DOF incidence, ascending (e, l)
    std::vector<int> dstart(nd + 1, 0), dinc(d.l2g().size());
    for (int k : d.l2g()) ++dstart[k + 1];
    for (int i = 0; i < nd; ++i) dstart[i + 1] += dstart[i];
    {
      std::vector<int> fill(dstart.begin(), dstart.end() - 1);
      for (size_t k = 0; k < d.l2g().size(); ++k) dinc[fill[d.l2g()[k]]++] = static_cast<int>(k);
    }
    const int *d_dstart = up(dstart), *d_dinc = up(dinc);
    // chunk of test elements: block buffer and strips within ~1 GB each
    const size_t row_blk = static_cast<size_t>(ne) * NL * NL * sizeof(S), row_strip = static_cast<size_t>(NL) * nd * sizeof(S);
    const size_t budget = size_t(1) << 30;
    const int nrow = static_cast<int>(std::max<size_t>(1, std::min<size_t>(ne, budget / std::max(row_blk, row_strip))));
    S* d_buf = static_cast<S*>(alloc(static_cast<size_t>(nrow) * row_blk));
    S* d_strip = static_cast<S*>(alloc(static_cast<size_t>(nrow) * row_strip));
    S* d_A = static_cast<S*>(alloc(static_cast<size_t>(nd) * nd * sizeof(S)));
    int* d_rows = static_cast<int*>(alloc(static_cast<size_t>(nd) * sizeof(int)));
    IGB_CUDA(cudaMemsetAsync(d_A, 0, static_cast<size_t>(nd) * nd * sizeof(S), st));
    const int per = std::max(1, 128 / (NC * nq));
    const size_t rsmem = static_cast<size_t>(per) * NC * nq * NL * sizeof(S);
    IGB_CUDA(cudaFuncSetAttribute(k_regular_dense<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    if (rsmem > 200 * 1024) throw std::invalid_argument("B200 dense: far quadrature order too large");
    KParams kp;
    kp.kr = kp4[0];
    kp.ki = kp4[1];
    kp.dwx = kp4[2];
    kp.dwy = kp4[3];
    for (int ea0 = 0; ea0 < ne; ea0 += nrow) {
      const int nr = std::min(nrow, ne - ea0);
      const long long npair = static_cast<long long>(nr) * ne;
      k_regular_dense<KT><<<static_cast<unsigned>((npair + per - 1) / per), 128, rsmem, st>>>(
          npair, per, ea0, ne, nq, d_cpts, d_cval, kp, reinterpret_cast<double*>(d_buf));
      for (int c = 1; c <= 3; ++c) {
        const long long tot = static_cast<long long>(items[c].ea.size()) * NL * NL;
        if (tot)
          k_dense_sing_place<S, NL><<<grid_for(tot, 256), 256, 0, st>>>(static_cast<int>(items[c].ea.size()), d_ia[c],
                                                                        d_ib[c], d_sblk[c], ea0, nr, ne, d_buf);
      }
      const long long ns_ = static_cast<long long>(nr) * NL * nd;
      k_dense_strip<S, NL><<<grid_for(ns_, 256), 256, 0, st>>>(nr, nd, ne, d_dstart, d_dinc, d_lsign, d_buf, d_strip);
      std::vector<int> rows;
      for (int e = ea0; e < ea0 + nr; ++e)
        for (int l = 0; l < NL; ++l) rows.push_back(d.l2g()[static_cast<size_t>(e) * NL + l]);
      std::sort(rows.begin(), rows.end());
      rows.erase(std::unique(rows.begin(), rows.end()), rows.end());
      IGB_CUDA(cudaMemcpyAsync(d_rows, rows.data(), rows.size() * sizeof(int), cudaMemcpyHostToDevice, st));
      const long long nrw = static_cast<long long>(rows.size()) * nd;
      k_dense_rows<S, NL><<<grid_for(nrw, 256), 256, 0, st>>>(static_cast<int>(rows.size()), d_rows, nd, d_dstart,
                                                              d_dinc, d_lsign, ea0, nr, d_strip, d_A);
      IGB_CUDA(cudaGetLastError());
      IGB_CUDA(cudaStreamSynchronize(st));  // the host row list is reused next chunk
    }
    IGB_CUDA(cudaMemcpyAsync(out, d_A, static_cast<size_t>(nd) * nd * sizeof(S), cudaMemcpyDeviceToHost, st));
    IGB_CUDA(cudaStreamSynchronize(st));
  } catch (...) {
    if (st) cudaStreamSynchronize(st);
    for (void* p : mem) cudaFree(p);
    if (st) cudaStreamDestroy(st);
    throw;
  }
  for (void* p : mem) cudaFree(p);
  cudaStreamDestroy(st);
}

void dense_assemble(const Discretization& d, int far_order, int sing_order, int device, double* out) {
  const int kind = d.kind();
  const int q = kind == kMaxwell ? d.degree() : d.scalar_degree();
  if (kind == kMaxwell && (q < 1 || q > 3)) throw std::invalid_argument("B200 dense: Maxwell degree > 3 not instantiated");
  if (kind != kMaxwell && (q < 0 || q > 4)) throw std::invalid_argument("B200 dense: scalar degree > 4 not instantiated");
  auto run = [&](auto kt) { dense_impl<decltype(kt)>(d, far_order, sing_order, device, out); };
  if (kind == kLaplace) {
    switch (q) {
      case 0: run(LapT<0>{}); break;
      case 1: run(LapT<1>{}); break;
      case 2: run(LapT<2>{}); break;
      case 3: run(LapT<3>{}); break;
      default: run(LapT<4>{}); break;
    }
  } else if (kind == kHelmholtz) {
    switch (q) {
      case 0: run(HelmT<0>{}); break;
      case 1: run(HelmT<1>{}); break;
      case 2: run(HelmT<2>{}); break;
      case 3: run(HelmT<3>{}); break;
      default: run(HelmT<4>{}); break;
    }
  } else {
    switch (q) {
      case 1: run(MaxT<1>{}); break;
      case 2: run(MaxT<2>{}); break;
      default: run(MaxT<3>{}); break;
    }
  }
}

}  // namespace igb
