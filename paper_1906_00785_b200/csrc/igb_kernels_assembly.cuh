// B200 (sm_100a) assembly kernels of the H2 operator: element quadrature
// caches + Chebyshev moments (h2.cpp:131-173, pair_integration.hpp:40-73),
// interpolation-node images (h2.cpp:182-196), far couplings (h2.cpp:218-229),
// regular near blocks (pair_integration.hpp:76-95), dense Galerkin blocks
// (assembly.cpp:16-53) and the Sauter-Schwab singular blocks batched by class
// (pair_integration.hpp:98-148, quadrature.cpp:82-199).  Included once, by
// igb_device.cu (the kernels are instantiated where H2Device launches them).
#pragma once

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
  return static_cast<size_t>(rs) * NL * NL + row_tile_off(cnt * NL, NL, la, (q - rs) * NL + lb);
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

// ------------------------------------------------- K3b: leaf blocks
// Element block of a leaf-level admissible pair (t, s):
//   B[la][lb] = sum_nu sum_mu mom_t[la][nu] K[nu][mu] mom_s[lb][mu],
// K[nu][mu] = G(|img_t[nu] - img_s[mu]|) -- what apply() computes for the pair
// through leaf moments, coupling and leaf transform (h2.cpp:281-290, 312-326,
// 359-371), assembled once.  One CTA per test element t: its moments stay in
// shared memory while the CTA walks the row's blocked pairs (K, then
// T = K mom_s^T, then B = mom_t T) and writes them into the row in the tiled
// block-row layout (row_tile_off; k: position among the row's blocked pairs).
template <int M, int NL>
__global__ void __launch_bounds__(128) k_leaf_blocks(int ne, const int* __restrict__ rs,
                                                     const int* __restrict__ node_s, int epp, int npp, int leaf_off,
                                                     const double* __restrict__ img, const double* __restrict__ mom,
                                                     double* __restrict__ blk) {
  constexpr int MM = M * M;
  __shared__ double Mt[NL * MM], Ms[NL * MM], K[MM * MM], T[MM * NL], it[3 * MM], is[3 * MM];
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= ne) return;
  const int r0 = rs[e], cnt = rs[e + 1] - r0;
  if (cnt == 0) return;
  const int t = (e / epp) * npp + leaf_off + e % epp;
  for (int i = tid; i < NL * MM; i += 128) Mt[i] = __ldg(mom + static_cast<size_t>(e) * NL * MM + i);
  for (int i = tid; i < 3 * MM; i += 128) it[i] = __ldg(img + static_cast<size_t>(t) * 3 * MM + i);
  double* out = blk + static_cast<size_t>(r0) * NL * NL;
  for (int kk = 0; kk < cnt; ++kk) {
    const int s = node_s[r0 + kk];
    if (s < 0) continue;  // a near block of the row (k_pack_sym_near)
    const int es = (s / npp) * epp + (s % npp - leaf_off);
    __syncthreads();  // the previous pair is done with Ms, is, T
    for (int i = tid; i < NL * MM; i += 128) Ms[i] = __ldg(mom + static_cast<size_t>(es) * NL * MM + i);
    for (int i = tid; i < 3 * MM; i += 128) is[i] = __ldg(img + static_cast<size_t>(s) * 3 * MM + i);
    __syncthreads();
    for (int i = tid; i < MM * MM; i += 128) {
      const int nu = i / MM, mu = i - nu * MM;
      const double d0 = it[3 * nu] - is[3 * mu], d1 = it[3 * nu + 1] - is[3 * mu + 1], d2 = it[3 * nu + 2] - is[3 * mu + 2];
      K[i] = kInv4Pi * rsqrt_nr(d0 * d0 + d1 * d1 + d2 * d2);
    }
    __syncthreads();
    for (int i = tid; i < MM * NL; i += 128) {  // T[nu][lb] = sum_mu K[nu][mu] Ms[lb][mu]
      const int nu = i / NL, lb = i - nu * NL;
      double a = 0.0;
#pragma unroll 5
      for (int mu = 0; mu < MM; ++mu) a = fma(K[nu * MM + mu], Ms[lb * MM + mu], a);
      T[i] = a;
    }
    __syncthreads();
    for (int i = tid; i < NL * NL; i += 128) {  // B[la][lb] = sum_nu Mt[la][nu] T[nu][lb]
      const int la = i / NL, lb = i - la * NL;
      double a = 0.0;
#pragma unroll 5
      for (int nu = 0; nu < MM; ++nu) a = fma(Mt[la * MM + nu], T[nu * NL + lb], a);
      out[row_tile_off(cnt * NL, NL, la, kk * NL + lb)] = a;
    }
  }
}

// Complex kinds: every leaf-level admissible pair as an element block
//   B = sum_c w_c mom_t,c K mom_s,c^T   (complex; the moments are real; channels
// c of the Maxwell EFIE share the scalar kernel K, the divergence channel carries
// the weight -1/kappa^2), so the matvec streams nl^2 scalars per ordered pair
// instead of evaluating m^4 complex kernels per unordered pair (c3: 81 against
// 4096) or streaming the stored coupling (c4: 2.3 KB against 65 KB).  One CTA
// per element t walks the row's pairs with s > t and writes B into row t and
// B^T into row s (the kernel is symmetric); rows are the ordered far rows of
// the leaf nodes.
template <class KT>
__global__ void __launch_bounds__(128) k_leaf_blocks_c(int ne, int m, const int* __restrict__ rs,
                                                       const int* __restrict__ far_rs, const int* __restrict__ far_b,
                                                       const int* __restrict__ upper_start, const int* __restrict__ trans,
                                                       int epp, int npp, int leaf_off, const double* __restrict__ img,
                                                       const double* __restrict__ mom, KParams kp,
                                                       typename KT::S* __restrict__ blk) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NCH = KT::NC;
  const int mm = m * m, rows = NCH * mm;
  extern __shared__ __align__(16) double cbsm[];
  double* Mt = cbsm;
  double* Ms = Mt + NL * rows;
  double* it = Ms + NL * rows;
  double* is = it + 3 * mm;
  S* K = reinterpret_cast<S*>(is + 3 * mm + ((NL * rows * 2 + 6 * mm) & 1));
  S* T = K + mm * mm;  // [c][nu][lb]
  const int e = blockIdx.x, tid = threadIdx.x;
  if (e >= ne) return;
  const int t = (e / epp) * npp + leaf_off + e % epp;
  const int q_lo = upper_start[t], q_hi = far_rs[t + 1];
  if (q_lo == q_hi) return;
  const int r0 = rs[e], cnt = rs[e + 1] - r0;
  const S wdiv = mk(kp.dwx, kp.dwy);
  for (int i = tid; i < NL * rows; i += 128) Mt[i] = __ldg(mom + static_cast<size_t>(e) * NL * rows + i);
  for (int i = tid; i < 3 * mm; i += 128) it[i] = __ldg(img + static_cast<size_t>(t) * 3 * mm + i);
  for (int q = q_lo; q < q_hi; ++q) {
    const int s = far_b[q];
    const int es = (s / npp) * epp + (s % npp - leaf_off);
    __syncthreads();
    for (int i = tid; i < NL * rows; i += 128) Ms[i] = __ldg(mom + static_cast<size_t>(es) * NL * rows + i);
    for (int i = tid; i < 3 * mm; i += 128) is[i] = __ldg(img + static_cast<size_t>(s) * 3 * mm + i);
    __syncthreads();
    for (int i = tid; i < mm * mm; i += 128) {
      const int nu = i / mm, mu = i - nu * mm;
      const double d0 = it[3 * nu] - is[3 * mu], d1 = it[3 * nu + 1] - is[3 * mu + 1], d2 = it[3 * nu + 2] - is[3 * mu + 2];
      K[i] = green_k<KT>(d0 * d0 + d1 * d1 + d2 * d2, kp);
    }
    __syncthreads();
    for (int i = tid; i < NCH * mm * NL; i += 128) {  // T_c[nu][lb] = sum_mu K[nu][mu] Ms[lb][c mm + mu]
      const int c = i / (mm * NL), r = i - c * mm * NL, nu = r / NL, lb = r - nu * NL;
      S a = zero<S>();
      for (int mu = 0; mu < mm; ++mu) fmac(a, K[nu * mm + mu], Ms[lb * rows + c * mm + mu]);
      if (NCH == 4 && c == 3) a = a * wdiv;
      T[i] = a;
    }
    __syncthreads();
    const int kk = q - far_rs[t];
    const int qt = trans[q], rs_s = rs[es], cnt_s = rs[es + 1] - rs_s, kk_s = qt - far_rs[s];
    for (int i = tid; i < NL * NL; i += 128) {  // B[la][lb] = sum_c sum_nu Mt[la][c mm + nu] T_c[nu][lb]
      const int la = i / NL, lb = i - la * NL;
      S a = zero<S>();
      for (int c = 0; c < NCH; ++c)
        for (int nu = 0; nu < mm; ++nu) fmac(a, T[(c * mm + nu) * NL + lb], Mt[la * rows + c * mm + nu]);
      blk[static_cast<size_t>(r0) * NL * NL + row_tile_off(cnt * NL, NL, la, kk * NL + lb)] = a;
      blk[static_cast<size_t>(rs_s) * NL * NL + row_tile_off(cnt_s * NL, NL, lb, kk_s * NL + la)] = a;
    }
  }
}

// near blocks (e, f), f >= e, copied into the block rows of the warp-specialised
// leaf kernel (position k of row e; the diagonal block halved: the row's own
// product and its transposed product each give half of it); one warp per block
template <int NL>
__global__ void __launch_bounds__(128) k_pack_sym_near(int n_pos, const int* __restrict__ slot_q,
                                                       const int* __restrict__ eb, const int* __restrict__ rs,
                                                       const int* __restrict__ near_a, const int* __restrict__ near_rs,
                                                       const double* __restrict__ near, double* __restrict__ blk) {
  const int k = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (k >= n_pos) return;
  const int q = slot_q[k];
  if (q < 0) return;
  const int e = near_a[q];
  const double scale = eb[k] == e ? 0.5 : 1.0;
  const int r0 = rs[e], len = (rs[e + 1] - r0) * NL;
  double* out = blk + static_cast<size_t>(r0) * NL * NL;
  for (int i = lane; i < NL * NL; i += 32) {
    const int la = i / NL, lb = i - la * NL;
    out[row_tile_off(len, NL, la, (k - r0) * NL + lb)] = scale * near[near_off(near_a, near_rs, q, la, lb, NL)];
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


}  // namespace dev
}  // namespace igb
