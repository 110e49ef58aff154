// B200 (sm_100a) kernels of the seven phases of H2Matrix::apply
// (h2.cpp:254-378): coefficient gather, leaf moments and upward transfer, the
// far field (column-stream symmetric kernels evaluating the couplings on the
// fly, the lane-tile kernel for m = 6, the warp-row complex kernel, the
// stored-coupling streams), transposed-slot sums, downward transfer, near-field
// rows (fused with the leaf far field on one GPU), leaf backward transform and
// the deterministic DOF gather.  Included once, by igb_device.cu.
#pragma once

#include "igb_kernels_assembly.cuh"

namespace igb {
namespace dev {

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
                            S* __restrict__ up, S* __restrict__ down, long long ndown,
                            S* __restrict__ coef_out) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx < ndown) down[idx] = zero<S>();
  if (idx >= static_cast<long long>(n_el) * rows) return;
  const int e = static_cast<int>(idx / rows), r = static_cast<int>(idx % rows);
  S acc = zero<S>(), mine = zero<S>();
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const int k = e * NL + l;
    const S c = x[l2g[k]] * sg[k];
    if (l == r) mine = c;
    fmac(acc, c, __ldg(mom + static_cast<size_t>(k) * rows + r));
  }
  if (coef_out != nullptr && r < NL) coef_out[e * NL + r] = mine;  // rows >= NL
  const int leaf = (e / epp) * npp + leaf_off + (e % epp);
  up[static_cast<size_t>(leaf) * rows + r] = acc;
}

// The same with one warp per element (real scalars; the warp-specialised graph):
// the element's moments [l][row] are staged in shared memory by coalesced loads
// and lane r sums its row in the same FMA order, so the results are bit-identical
// to k_leaf_up_x; also writes the element coefficients and zeroes down.
template <int NL>
__global__ void __launch_bounds__(256) k_leaf_up_w(int n_el, int rows, int epp, int npp, int leaf_off,
                                                   const double* __restrict__ mom, const double* __restrict__ x,
                                                   const int* __restrict__ l2g, const double* __restrict__ sg,
                                                   double* __restrict__ up, double* __restrict__ down, long long ndown,
                                                   double* __restrict__ coef_out) {
  pdl_entry();
  constexpr int MAXR = 32;  // rows <= 32 (m <= 5)
  __shared__ double sh[8][NL * MAXR + NL];
  const long long tid = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const long long total = static_cast<long long>(gridDim.x) * blockDim.x;
  for (long long i = tid; i < ndown; i += total) down[i] = 0.0;
  const int e = static_cast<int>(tid >> 5), lane = threadIdx.x & 31;
  if (e >= n_el) return;
  double* ms = sh[threadIdx.x >> 5];
  double* cs = ms + NL * MAXR;
  const double* me = mom + static_cast<size_t>(e) * NL * rows;
  for (int i = lane; i < NL * rows; i += 32) ms[i] = __ldg(me + i);
  if (lane < NL) {
    const int k = e * NL + lane;
    const double c = x[l2g[k]] * sg[k];
    cs[lane] = c;
    coef_out[k] = c;
  }
  __syncwarp();
  if (lane < rows) {
    double acc = 0.0;
#pragma unroll
    for (int l = 0; l < NL; ++l) acc = fma(cs[l], ms[l * rows + lane], acc);
    const int leaf = (e / epp) * npp + leaf_off + (e % epp);
    up[static_cast<size_t>(leaf) * rows + lane] = acc;
  }
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
// far_end[t]: end of the target's evaluated upper pairs -- its row end
// (far_rs + 1) or, for leaf targets with blocked pairs (LeafBlocks), before them
template <int M, int C, bool LIST = false>
__device__ __forceinline__ void far_col_body(int t, int lane, double* __restrict__ sh,
                                             const int* __restrict__ upper_start, const int* __restrict__ far_end,
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
  const int ncol = ((LIST ? col_q1 : far_end[t]) - q0) * MM;
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
                                                      const int* __restrict__ far_end, const int* __restrict__ far_b,
                                                      const int* __restrict__ trans, const double* __restrict__ img,
                                                      const double* __restrict__ up, double* __restrict__ down,
                                                      double* __restrict__ slot) {
  __shared__ __align__(16) double sh[8][(5 * M * M + 1) / 2 * 2];
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (warp >= n_targets) return;
  far_col_body<M, C>(targets[warp], threadIdx.x & 31, sh[threadIdx.x >> 5], upper_start, far_end, far_b, trans, img,
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

// the same over an explicit list of slots per row (leaf blocks: only the pairs
// the far kernels evaluate have a slot to add), ascending
__global__ void k_far_lower_list(int n_nodes, int mm, const int* __restrict__ low_rs, const int* __restrict__ low_q,
                                 const double* __restrict__ slot, double* __restrict__ down, int rows, int npp,
                                 int leaf_off) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_nodes) * mm) return;
  const int s = static_cast<int>(idx / mm), nu = static_cast<int>(idx % mm);
  if (rows != 0 && ((s % npp >= leaf_off) != (rows == 1))) return;
  const int k0 = low_rs[s], k1 = low_rs[s + 1];
  if (k0 == k1) return;
  double acc = down[idx];
#pragma unroll 4
  for (int k = k0; k < k1; ++k) acc += __ldcs(slot + static_cast<size_t>(__ldg(low_q + k)) * mm + nu);
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
// streaming its contiguous row (tiled block-row layout, row_tile_off)
// FROM_X: coefficients gathered inline from x (l2g, signs) instead of coef
// SYM (leaf blocks, below): the row's blocks are those of unordered pairs
// (e, f), f > e; lane j = column (k, lb) also forms the transposed product
// sum_la blk[la][j] c_e[la] -- a lane-local sum -- into tslot[row start NL + j],
// which the leaf transform of element f adds.  xt: c_e in shared memory.
template <class S, int NL, bool FROM_X, bool SYM = false>
__device__ __forceinline__ void near_row_seg(S (&acc)[NL], int e, int lane, const int* __restrict__ near_rs,
                                             const int* __restrict__ near_b, const S* __restrict__ blk,
                                             const S* __restrict__ coef, const int* __restrict__ l2g,
                                             const double* __restrict__ sg, S* __restrict__ tslot = nullptr,
                                             S* __restrict__ xt = nullptr) {
  auto cf = [&](int k) -> S {
    if constexpr (FROM_X) return coef[l2g[k]] * sg[k];
    else return coef[k];
  };
  const int rs = near_rs[e], cnt = near_rs[e + 1] - rs;
  if (SYM && cnt == 0) return;
  const int len = cnt * NL;
  const S* base = blk + static_cast<size_t>(rs) * NL * NL;
  if constexpr (SYM) {
    __syncwarp();
    if (lane < NL) xt[lane] = cf(e * NL + lane);
    __syncwarp();
  }
  constexpr int U = (NL <= 9) ? 4 : 2;
  static_assert(kRowTile % 32 == 0, "a lane's columns of one step lie in whole tiles");
  int j = lane;
  for (; j + 32 * (U - 1) < len; j += 32 * U) {
    S xv[U], ps[U];
    const S* tb[U];  // column j + 32 u of its tile (row_tile_off): tile base + la * tile width
    int wt[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int jj = j + 32 * u, k = jj / NL, lb = jj - k * NL;
      xv[u] = cf(near_b[rs + k] * NL + lb);
      ps[u] = zero<S>();
      const int t0 = jj & ~(kRowTile - 1);
      wt[u] = min(kRowTile, len - t0);
      tb[u] = base + static_cast<size_t>(t0) * NL + (jj - t0);
    }
#pragma unroll
    for (int la = 0; la < NL; ++la) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const S v = ldg_s(tb[u] + la * wt[u]);
        fmac(acc[la], v, xv[u]);
        if constexpr (SYM) fmac(ps[u], v, xt[la]);
      }
    }
    if constexpr (SYM) {
#pragma unroll
      for (int u = 0; u < U; ++u) tslot[static_cast<size_t>(rs) * NL + j + 32 * u] = ps[u];
    }
  }
  for (; j < len; j += 32) {
    const int k = j / NL, lb = j - k * NL;
    const S xv = cf(near_b[rs + k] * NL + lb);
    S ps = zero<S>();
    const int t0 = j & ~(kRowTile - 1), wt = min(kRowTile, len - t0);
    const S* tb = base + static_cast<size_t>(t0) * NL + (j - t0);
#pragma unroll
    for (int la = 0; la < NL; ++la) {
      const S v = ldg_s(tb + la * wt);
      fmac(acc[la], v, xv);
      if constexpr (SYM) fmac(ps, v, xt[la]);
    }
    if constexpr (SYM) tslot[static_cast<size_t>(rs) * NL + j] = ps;
  }
}
// ACC: add to rows_out (a second set of block rows of the same elements)
template <class S, int NL, bool FROM_X, bool ACC = false>
__device__ __forceinline__ void near_row(int e, int lane, const int* __restrict__ near_rs,
                                         const int* __restrict__ near_b, const S* __restrict__ blk,
                                         const S* __restrict__ coef, S* __restrict__ rows_out,
                                         const int* __restrict__ l2g, const double* __restrict__ sg) {
  S acc[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) acc[l] = zero<S>();
  near_row_seg<S, NL, FROM_X>(acc, e, lane, near_rs, near_b, blk, coef, l2g, sg);
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const S a = warp_sum(acc[l]);
    if (lane == 0) {
      if constexpr (ACC) rows_out[static_cast<size_t>(e) * NL + l] = rows_out[static_cast<size_t>(e) * NL + l] + a;
      else rows_out[static_cast<size_t>(e) * NL + l] = a;
    }
  }
}
// the leaf blocks of the complex kinds (k_leaf_blocks_c): added to the near rows
template <class S, int NL>
__global__ void __launch_bounds__(256) k_block_rows_acc(int ne, const int* __restrict__ rs, const int* __restrict__ eb,
                                                        const S* __restrict__ blk, const S* __restrict__ coef,
                                                        S* __restrict__ rows_out) {
  const int e = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (e >= ne) return;
  if (rs[e] == rs[e + 1]) return;
  near_row<S, NL, false, true>(e, threadIdx.x & 31, rs, eb, blk, coef, rows_out, nullptr, nullptr);
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
// LeafBlocks: the last upper pairs of every leaf target are not evaluated but
// stored as element blocks M_t K M_s^T (k_leaf_blocks) and streamed like near
// blocks, each once for both directions (near_row_seg SYM) -- the FP64-bound
// kernel leaves HBM idle, so part of its work moves there.
struct LeafBlocks {
  const int* far_end;   // per node: end of the evaluated upper pairs
  const int* rs;        // per element: first blocked pair (CSR), null: none
  const int* eb;        // source element of each blocked pair
  const double* blk;    // element rows, tiled block-row layout
  double* tslot;        // transposed products [pair][lb]
};
template <int M, int NL, int MINB, int C>
__global__ void __launch_bounds__(256, MINB) k_far_col_near(
    int n_fine, const int* __restrict__ fine, int n_rest, const int* __restrict__ rest, int epp, int npp,
    int leaf_off, const int* __restrict__ upper_start, LeafBlocks lb,
    const int* __restrict__ far_b, const int* __restrict__ trans, const double* __restrict__ img,
    const double* __restrict__ up, double* __restrict__ down, double* __restrict__ slot,
    const unsigned char* __restrict__ /*owned: single GPU*/, const int* __restrict__ near_rs,
    const int* __restrict__ near_b, const double* __restrict__ blk, const double* __restrict__ x,
    double* __restrict__ rows_out, const int* __restrict__ l2g, const double* __restrict__ sg) {
  __shared__ __align__(16) double sh[8][(5 * M * M + 1) / 2 * 2];
  static_assert(5 * M * M >= NL, "shared slab holds the element's coefficients");
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  int e;
  if (warp < n_fine) {
    const int t = fine[warp];
    far_col_body<M, C>(t, lane, sh[threadIdx.x >> 5], upper_start, lb.far_end, far_b, trans, img, up, down, slot);
    e = (t / npp) * epp + (t % npp - leaf_off);
  } else if (warp < n_fine + n_rest) {
    e = rest[warp - n_fine];
  } else {
    return;
  }
  double acc[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) acc[l] = 0.0;
  near_row_seg<double, NL, true>(acc, e, lane, near_rs, near_b, blk, x, l2g, sg);
  if (lb.rs != nullptr)
    near_row_seg<double, NL, true, true>(acc, e, lane, lb.rs, lb.eb, lb.blk, x, l2g, sg, lb.tslot,
                                         sh[threadIdx.x >> 5]);
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const double a = warp_sum(acc[l]);
    if (lane == 0) rows_out[static_cast<size_t>(e) * NL + l] = a;
  }
}

// ---- warp-specialised leaf kernel (single GPU, NL = 16) ------------------
// One persistent 512-thread CTA per SM: twelve far warps run the column-stream
// far field over the leaf targets while four stream warps move the near rows
// and the leaf blocks through a shared-memory ring with bulk asynchronous copies
// (cp.async.bulk + mbarrier, no registers in flight), so the FP64 pipe and HBM
// are busy at the same time on every SM -- inside one warp the two phases only
// alternate.  A slice = one tile of a block row (row_tile_off: kRowTile columns
// x NL test functions, contiguous: one copy) plus the coefficient vectors of
// its blocks' source elements (one copy each).
namespace ws {
// 12 + 4 warps, 2 stages of one 17 KB tile each per stream warp (c5, kernel ms:
// 6.33; 3 stages 6.42; 11 + 5 warps 6.54, 10 + 6 warps 7.09; with the leaf far
// field still evaluated by half: 13 + 3 warps 6.41, 14 + 2 warps 8.33 against 5.84).
// With every leaf pair a block the split no longer matters (12 + 4: 6.20, 11 + 5:
// 6.22, 10 + 6: 6.37, 8 + 8 with one stage: 6.23): the kernel moves 36-39 GB of
// DRAM traffic at 6.1-6.3 TB/s, 93-96 % of the measured HBM peak.
constexpr int kStreamWarps = 4, kFarWarps = 16 - kStreamWarps, kStages = 2;
__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }
__device__ __forceinline__ void mbar_init(unsigned long long* bar, int count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  unsigned ok = 0;
  const unsigned a = smem_u32(bar);
  while (!ok)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(ok)
        : "r"(a), "r"(parity)
        : "memory");
}
// streamed once: evict-first in L2 (the far warps' node images and moments stay)
__device__ __forceinline__ unsigned long long policy_evict_first() {
  unsigned long long p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ void bulk_g2s_hint(void* dst, const void* src, unsigned bytes, unsigned long long* bar,
                                              unsigned long long policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 16 B per lane, completion counted by the stage's mbarrier
__device__ __forceinline__ void cp16_g2s(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_arrive(unsigned long long* bar) {
  asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(bar)) : "memory");
}
template <int M, int NL>
struct Layout {
  static constexpr int SLAB = (5 * M * M + 1) / 2 * 2;             // far warp: target rows + moments
  static constexpr int STAGE = (NL + 1) * kRowTile + NL;           // stream stage: tile [NL][w] + coefficients [w] + the row element's own [NL]
  static constexpr int FAR0 = 0;
  static constexpr int RING0 = (kFarWarps * SLAB + 15) / 16 * 16;  // doubles, 128 B aligned
  static constexpr int XT0 = RING0 + kStreamWarps * kStages * STAGE;
  static constexpr int DESC0 = XT0 + kStreamWarps * NL;            // int4 per stage
  static constexpr int BAR0 = DESC0 + kStreamWarps * kStages * 2;
  static constexpr int TOTAL = BAR0 + kStreamWarps * kStages;
  static constexpr size_t BYTES = static_cast<size_t>(TOTAL) * 8;
};
}  // namespace ws

template <int M, int NL, int C>
__global__ void __launch_bounds__(32 * (ws::kFarWarps + ws::kStreamWarps), 1) k_leaf_ws(
    int n_fine, const int* __restrict__ fine, int ne, const int* __restrict__ upper_start, LeafBlocks lb,
    const int* __restrict__ far_b, const int* __restrict__ trans, const double* __restrict__ img,
    const double* __restrict__ up, double* __restrict__ down, double* __restrict__ slot,
    const int* __restrict__ near_rs, const int* __restrict__ near_b, const double* __restrict__ blk,
    const double* __restrict__ coef, double* __restrict__ rows_out) {
  using LY = ws::Layout<M, NL>;
  constexpr int W = kRowTile, NS = ws::kStages;
  static_assert(NL % 2 == 0 && W % NL == 0 && W % 64 == 0, "16 B coefficient pairs inside one block");
  extern __shared__ __align__(128) double wsm[];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < ws::kFarWarps) {  // ---- far warps
    double* sh = wsm + LY::FAR0 + warp * LY::SLAB;
    for (int i = blockIdx.x * ws::kFarWarps + warp; i < n_fine; i += gridDim.x * ws::kFarWarps) {
      far_col_body<M, C>(fine[i], lane, sh, upper_start, lb.far_end, far_b, trans, img, up, down, slot);
      __syncwarp();  // the slab is rewritten for the next target
    }
    return;
  }
  // ---- stream warps
  const int sw = warp - ws::kFarWarps;
  double* ring = wsm + LY::RING0 + sw * NS * LY::STAGE;
  double* xt = wsm + LY::XT0 + sw * NL;
  int4* desc = reinterpret_cast<int4*>(wsm + LY::DESC0) + sw * NS;
  unsigned long long* bar = reinterpret_cast<unsigned long long*>(wsm + LY::BAR0) + sw * NS;
  if (lane == 0) {
    for (int i = 0; i < NS; ++i) ws::mbar_init(bar + i, 33);  // expect_tx arrive + one per lane (coefficients)
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();
  // slice generator (warp-uniform): elements e = first, first + stride, ...;
  // segment 0 the near row, segment 1 the leaf blocks of e.  The row extents of
  // the next element are read one element ahead.
  const int stride = gridDim.x * ws::kStreamWarps;
  int g_e = blockIdx.x * ws::kStreamWarps + sw, g_seg = 0, g_j0 = 0, g_rs = 0, g_len = 0, g_len1 = 0, g_rs1 = 0;
  int n_rs = 0, n_re = 0, n_rs1 = 0, n_re1 = 0;
  auto fetch_item = [&](int e) {
    if (e < ne) {
      n_rs = near_rs ? near_rs[e] : 0;  // null: the near field is part of the block rows
      n_re = near_rs ? near_rs[e + 1] : 0;
      n_rs1 = lb.rs ? lb.rs[e] : 0;
      n_re1 = lb.rs ? lb.rs[e + 1] : 0;
    }
  };
  auto load_item = [&]() {  // element g_e from the prefetched extents; prefetch the next
    g_rs = n_rs;
    g_len = (n_re - n_rs) * NL;
    g_rs1 = n_rs1;
    g_len1 = (n_re1 - n_rs1) * NL;
    g_seg = g_len > 0 ? 0 : 1;
    g_j0 = 0;
    fetch_item(g_e + stride);
  };
  fetch_item(g_e);
  if (g_e < ne) load_item();
  const unsigned long long pol = ws::policy_evict_first();
  // source elements of the blocks holding this lane's coefficient pairs (columns
  // 2 lane + 64 h + {0, 1}) of the current slice, read one slice ahead
  constexpr int H = W / 64;
  int pf_e[H];
#pragma unroll
  for (int h = 0; h < H; ++h) pf_e[h] = 0;
  auto prefetch_src = [&]() {
    if (g_e >= ne) return;
    const int rs = g_seg ? g_rs1 : g_rs, len = g_seg ? g_len1 : g_len;
    const int w = min(W, len - g_j0);
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int c = 2 * lane + 64 * h;
      if (c < w) pf_e[h] = (g_seg ? lb.eb : near_b)[rs + (g_j0 + c) / NL];
    }
  };
  prefetch_src();
  // issue the generator's current slice into stage s and advance: the tile as one
  // bulk copy (lane 0), the coefficients as one 16 B asynchronous copy per lane
  auto issue = [&](int s) {
    const int rs = g_seg ? g_rs1 : g_rs, len = g_seg ? g_len1 : g_len;
    const int w = min(W, len - g_j0);
    const bool last_seg = g_seg == 1 || g_len1 == 0;
    const bool first = g_j0 == 0 && (g_seg == 0 || g_len == 0), last = last_seg && g_j0 + w >= len;
    double* st = ring + s * LY::STAGE;
#pragma unroll
    for (int h = 0; h < H; ++h) {
      const int c = 2 * lane + 64 * h;
      if (c < w) ws::cp16_g2s(st + NL * W + c, coef + static_cast<size_t>(pf_e[h]) * NL + (g_j0 + c) % NL);
    }
    // first slice of a row's blocks: the row element's own coefficients ride along
    if (g_seg == 1 && g_j0 == 0 && 2 * lane < NL)
      ws::cp16_g2s(st + (NL + 1) * W + 2 * lane, coef + static_cast<size_t>(g_e) * NL + 2 * lane);
    ws::cp_arrive(bar + s);
    if (lane == 0) {
      desc[s] = make_int4(g_e, rs * NL + g_j0, w, (first ? 1 : 0) | (last ? 2 : 0) | (g_seg ? 4 : 0) | ((g_seg && g_j0 == 0) ? 8 : 0));
      ws::mbar_expect_tx(bar + s, static_cast<unsigned>(w) * NL * 8u);
      const double* base = (g_seg ? lb.blk : blk) + static_cast<size_t>(rs) * NL * NL;
      ws::bulk_g2s_hint(st, base + static_cast<size_t>(g_j0) * NL, static_cast<unsigned>(w) * NL * 8u, bar + s, pol);
    }
    __syncwarp();
    g_j0 += w;
    if (g_j0 >= len) {
      g_j0 = 0;
      if (g_seg == 0 && g_len1 > 0) {
        g_seg = 1;
      } else {
        g_e += stride;
        if (g_e < ne) load_item();
      }
    }
    prefetch_src();
  };
  int issued = 0, consumed = 0;
  for (; issued < NS && g_e < ne; ++issued) issue(issued);
  double acc[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) acc[l] = 0.0;
  while (consumed < issued) {
    const int s = consumed % NS;
    ws::mbar_wait(bar + s, (consumed / NS) & 1);
    const int4 d = desc[s];
    const double* st = ring + s * LY::STAGE;
    if (d.w & 8) {  // first slice of the row's blocks: this element's coefficients
      if (lane < NL) xt[lane] = st[(NL + 1) * W + lane];
      __syncwarp();
    }
    if (d.w & 1) {
#pragma unroll
      for (int l = 0; l < NL; ++l) acc[l] = 0.0;
    }
    {
#pragma unroll
      for (int h = 0; h < H; ++h) {  // columns c, c + 1 of the tile [la][w]: 16 B loads
        const int c = 2 * lane + 64 * h;
        if (c < d.z) {
          const double2 xv = *reinterpret_cast<const double2*>(st + NL * W + c);
          const double* tc = st + c;
          if (d.w & 4) {
            double2 ps = make_double2(0.0, 0.0);
#pragma unroll
            for (int la = 0; la < NL; ++la) {
              const double2 v = *reinterpret_cast<const double2*>(tc + la * d.z);
              acc[la] = fma(v.x, xv.x, acc[la]);
              acc[la] = fma(v.y, xv.y, acc[la]);
              const double t = xt[la];
              ps.x = fma(v.x, t, ps.x);
              ps.y = fma(v.y, t, ps.y);
            }
            *reinterpret_cast<double2*>(lb.tslot + static_cast<size_t>(d.y) + c) = ps;
          } else {
#pragma unroll
            for (int la = 0; la < NL; ++la) {
              const double2 v = *reinterpret_cast<const double2*>(tc + la * d.z);
              acc[la] = fma(v.x, xv.x, acc[la]);
              acc[la] = fma(v.y, xv.y, acc[la]);
            }
          }
        }
      }
    }
    if (d.w & 2) {  // row sums over the lanes: reduce-scatter, lane l < NL ends with function l
      col_reduce_rows<NL>(acc, lane);
      if (lane < NL) rows_out[static_cast<size_t>(d.x) * NL + lane] = acc[0];
    }
    __syncwarp();  // every lane is done with stage s (and its descriptor)
    ++consumed;
    if (g_e < ne) {  // refill the stage just consumed
      issue(s);
      ++issued;
    }
  }
}

// leaf backward transform moments^T down + near rows (h2.cpp:359-371); one
// thread per (owned element, local function)
template <class S, int NL>
__global__ void __launch_bounds__(256) k_leaf_down(int n_el, const int* __restrict__ el, int rows, int epp, int npp,
                                                   int leaf_off, const double* __restrict__ mom,
                                                   const S* __restrict__ down, const S* __restrict__ near_rows,
                                                   S* __restrict__ loc, const int* __restrict__ in_rs = nullptr,
                                                   const int* __restrict__ in_k = nullptr,
                                                   const S* __restrict__ tslot = nullptr) {
  pdl_entry();
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (idx >= static_cast<long long>(n_el) * NL) return;
  const int i = static_cast<int>(idx / NL), l = static_cast<int>(idx % NL);
  const int e = el[i];
  const int leaf = (e / epp) * npp + leaf_off + (e % epp);
  const S* dn = down + static_cast<size_t>(leaf) * rows;
  const double* mc = mom + (static_cast<size_t>(e) * NL + l) * rows;
  S acc = zero<S>();
  if (in_rs != nullptr)  // leaf blocks: transposed products of the pairs (f, e), f < e, in fixed order
    for (int j = in_rs[e]; j < in_rs[e + 1]; ++j) acc = acc + tslot[static_cast<size_t>(in_k[j]) * NL + l];
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
}  // namespace igb
