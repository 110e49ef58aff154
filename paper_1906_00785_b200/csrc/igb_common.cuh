// Shared sm_100a device helpers: FP64 / complex scalars, Green's functions
// (operators.hpp:16-20), rational geometry jets on the power-basis cells, and
// the B-spline / Piola shape functions (spaces.cpp:257-307).
#pragma once

#include <cuda_runtime.h>

#include <cstdio>
#include <stdexcept>
#include <string>

#define IGB_CUDA(x)                                                                          \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess)                                                                   \
      throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_) + " (" + \
                               #x + ")");                                                    \
  } while (0)

namespace igb {
namespace dev {

// Block rows (near field, leaf blocks): the row of a test element holds its
// blocks as columns j = k NL + lb (k-th block, trial function lb) for each test
// function la.  Tiled layout: tiles of kRowTile columns, each tile stored
// [la][column] contiguously -- a warp streams one tile per step and a tile is
// one contiguous piece for a bulk copy.
constexpr int kRowTile = 128;
__host__ __device__ inline size_t row_tile_off(int len, int nl, int la, int j) {
  const int t0 = (j / kRowTile) * kRowTile;
  const int wt = len - t0 < kRowTile ? len - t0 : kRowTile;
  return static_cast<size_t>(t0) * nl + static_cast<size_t>(la) * wt + (j - t0);
}
constexpr double kInv4Pi = 0.079577471545947667884;  // 1 / (4 pi)
constexpr int kCellStride = 104;                       // 100 coefficients + u0, v0 (+pad)

// ------------------------------------------------------------ scalars
struct __align__(16) cd {
  double x, y;
};
__host__ __device__ __forceinline__ cd mk(double a, double b) {
  cd r;
  r.x = a;
  r.y = b;
  return r;
}
template <class S>
__host__ __device__ __forceinline__ S mk_s(double re, double im);
template <>
__host__ __device__ __forceinline__ double mk_s<double>(double re, double) { return re; }
template <>
__host__ __device__ __forceinline__ cd mk_s<cd>(double re, double im) { return mk(re, im); }
template <class S>
__device__ __forceinline__ S zero();
template <>
__device__ __forceinline__ double zero<double>() { return 0.0; }
template <>
__device__ __forceinline__ cd zero<cd>() { return mk(0.0, 0.0); }

__device__ __forceinline__ double operator_add(double a, double b) { return a + b; }
__device__ __forceinline__ cd operator+(cd a, cd b) { return mk(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ cd operator*(cd a, cd b) { return mk(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x); }
__device__ __forceinline__ cd operator*(cd a, double b) { return mk(a.x * b, a.y * b); }
__device__ __forceinline__ cd operator*(double b, cd a) { return mk(a.x * b, a.y * b); }

__device__ __forceinline__ void fmac(double& acc, double a, double b) { acc = fma(a, b, acc); }
__device__ __forceinline__ void fmac(cd& acc, cd a, double b) {
  acc.x = fma(a.x, b, acc.x);
  acc.y = fma(a.y, b, acc.y);
}
__device__ __forceinline__ void fmac(cd& acc, double a, cd b) { fmac(acc, b, a); }
__device__ __forceinline__ void fmac(cd& acc, cd a, cd b) {
  acc.x = fma(a.x, b.x, acc.x);
  acc.x = fma(-a.y, b.y, acc.x);
  acc.y = fma(a.x, b.y, acc.y);
  acc.y = fma(a.y, b.x, acc.y);
}
__device__ __forceinline__ double shfl_down(double v, int o) { return __shfl_down_sync(0xffffffffu, v, o); }
__device__ __forceinline__ cd shfl_down(cd v, int o) {
  return mk(__shfl_down_sync(0xffffffffu, v.x, o), __shfl_down_sync(0xffffffffu, v.y, o));
}
__device__ __forceinline__ double shfl_idx(double v, int src) { return __shfl_sync(0xffffffffu, v, src); }
__device__ __forceinline__ cd shfl_idx(cd v, int src) {
  return mk(__shfl_sync(0xffffffffu, v.x, src), __shfl_sync(0xffffffffu, v.y, src));
}
__device__ __forceinline__ double shfl_xor(double v, int o) { return __shfl_xor_sync(0xffffffffu, v, o); }
__device__ __forceinline__ cd shfl_xor(cd v, int o) {
  return mk(__shfl_xor_sync(0xffffffffu, v.x, o), __shfl_xor_sync(0xffffffffu, v.y, o));
}
// programmatic dependent launch: allow the next kernel of the stream to launch,
// then wait for this kernel's predecessors (no-ops when launched without PDL)
__device__ __forceinline__ void pdl_entry() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ double ldg_s(const double* p) { return __ldg(p); }
__device__ __forceinline__ cd ldg_s(const cd* p) {
  const double2 v = __ldg(reinterpret_cast<const double2*>(p));
  return mk(v.x, v.y);
}
template <class S>
__device__ __forceinline__ S warp_sum(S v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = v + shfl_down(v, o);
  return v;  // valid in lane 0
}

// ------------------------------------------------------ kernel traits
struct KParams {
  double kr, ki;      // wavenumber
  double dwx, dwy;    // -1/kappa^2 (Maxwell divergence weight)
};
template <int Q_>
struct LapT {
  using S = double;
  static constexpr int KIND = 0, Q = Q_, NL = (Q_ + 1) * (Q_ + 1), NC = 1, CHUNK = 128;
  static constexpr int TS = Q_ + 1;                  // accumulation tile side
  static constexpr int TABN = 2 * (Q_ + 1) * (Q_ + 1);  // per element: u and v tables
};
template <int Q_>
struct HelmT {
  using S = cd;
  static constexpr int KIND = 1, Q = Q_, NL = (Q_ + 1) * (Q_ + 1), NC = 1, CHUNK = 128;
  static constexpr int TS = Q_ + 1;
  static constexpr int TABN = 2 * (Q_ + 1) * (Q_ + 1);
};
template <int P_>
struct MaxT {
  using S = cd;
  static constexpr int KIND = 2, Q = P_, NL = 2 * (P_ + 1) * P_, NC = 4, CHUNK = 64;
  static constexpr int TS = (NL % 4 == 0) ? 4 : 2;
  // per element: p-tables (u, v) of (P+1)^2 and q-tables (u, v) of P^2, padded even
  static constexpr int TABN = ((2 * (P_ + 1) * (P_ + 1) + 2 * P_ * P_) + 1) / 2 * 2;
};

// Green's functions (operators.hpp:16-20), distance clamped as in
// pair_integration.hpp:18,118
// Branch-free FP64 reciprocal square root for normal positive inputs:
// MUFU.RSQ64H seed (rsqrt.approx.ftz.f64, rel. err < 2^-22) + 2 Newton steps.
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y0;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(x));
  // one cubic (Householder) step: y = y0 (1 + e/2 + 3e^2/8), e = 1 - x y0^2
  const double e = fma(-x * y0, y0, 1.0);
  return fma(y0 * e, fma(0.375, e, 0.5), y0);
}

// G(max(r, 1e-14)) (operators.hpp:16-20, pair_integration.hpp:22-28); 1/r from
// the refined reciprocal square root (~1 ulp), r = r^2 / r
__device__ __forceinline__ double green(double r2, const KParams&, double) {
  return rsqrt_nr(fmax(r2, 1e-28)) * kInv4Pi;
}
__device__ __forceinline__ cd green_c(double r2, const KParams& kp) {
  const double r2c = fmax(r2, 1e-28);
  const double ir = rsqrt_nr(r2c), r = r2c * ir;
  double s, c;
  sincos(kp.kr * r, &s, &c);
  double a = kInv4Pi * ir;
  if (kp.ki != 0.0) a *= exp(kp.ki * r);
  return mk(a * c, -a * s);
}
// sin and cos for the far field: x - k pi/2 by two FMAs with a two-part pi/2
// (k = rint(2x/pi)), then the fdlibm kernel polynomials on [-pi/4, pi/4]
// (__kernel_sin / __kernel_cos coefficients, error < 2^-58 there) and the
// quadrant swap; libdevice sincos beyond |x| = 1e5
__device__ __forceinline__ void sincos_far(double x, double* sn, double* cs) {
  if (fabs(x) > 1e5) {
    sincos(x, sn, cs);
    return;
  }
  const double k = rint(x * 0.63661977236758134308);
  const double y = fma(-k, 6.12323399573676603587e-17, fma(-k, 1.57079632679489655800e+00, x));
  const double z = y * y;
  const double ps = fma(fma(fma(fma(fma(1.58969099521155010221e-10, z, -2.50507602534068634195e-08), z,
                                    2.75573137070700676789e-06), z, -1.98412698298579493134e-04), z,
                            8.33333333332248946124e-03), z, -1.66666666666666324348e-01);
  const double pc = fma(fma(fma(fma(fma(-1.13596475577881948265e-11, z, 2.08757232129817482790e-09), z,
                                    -2.75573143513906633035e-07), z, 2.48015872894767294178e-05), z,
                            -1.38888888888741095749e-03), z, 4.16666666666666019037e-02);
  const double s0 = fma(y * z, ps, y);
  const double c0 = fma(z * z, pc, fma(-0.5, z, 1.0));
  const int q = __double2int_rn(k);
  double s = (q & 1) ? c0 : s0, c = (q & 1) ? s0 : c0;
  if (q & 2) s = -s;
  if ((q + 1) & 2) c = -c;
  *sn = s;
  *cs = c;
}
// Green's function for the far field (admissible pairs, r > 0).  Laplace: 1/r
// from the MUFU estimate and one Newton step (relative error ~1e-13, far below
// the interpolation error).  Complex kinds: the cubic refinement (~1 ulp: the
// phase kappa r amplifies an error in r) and the reduced-range sincos above.
template <class KT>
__device__ __forceinline__ typename KT::S green_far(double r2, const KParams& kp) {
  if constexpr (KT::KIND == 0) {
    double y0;
    asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(r2));
    return (0.5 * kInv4Pi) * (y0 * fma(-r2 * y0, y0, 3.0));
  } else {
    const double ir = rsqrt_nr(r2), r = r2 * ir;
    double s, c;
    sincos_far(kp.kr * r, &s, &c);
    double a = kInv4Pi * ir;
    if (kp.ki != 0.0) a *= exp(kp.ki * r);
    return mk(a * c, -a * s);
  }
}
template <class KT>
__device__ __forceinline__ typename KT::S green_k(double r2, const KParams& kp) {
  if constexpr (KT::KIND == 0)
    return green(r2, kp, 0.0);
  else
    return green_c(r2, kp);
}

// -------------------------------------------------------- geometry jet
// cf: [c][j][i] (stride 5 / 25), homogeneous (wx, wy, wz, w) in (s, t)
template <int D>
__device__ __forceinline__ void jet(const double* __restrict__ cf, double s, double t, double x[3],
                                    double du[3], double dv[3]) {
  double N[4], Ns[4], Nt[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* p = cf + c * 25;
    double n = 0.0, ns = 0.0, nt = 0.0;
#pragma unroll
    for (int j = D; j >= 0; --j) {
      double r = p[j * 5 + D], rp = 0.0;
#pragma unroll
      for (int i = D - 1; i >= 0; --i) {
        rp = fma(rp, s, r);
        r = fma(r, s, p[j * 5 + i]);
      }
      nt = fma(nt, t, n);
      n = fma(n, t, r);
      ns = fma(ns, t, rp);
    }
    N[c] = n;
    Ns[c] = ns;
    Nt[c] = nt;
  }
  const double iw = 1.0 / N[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    x[k] = N[k] * iw;
    du[k] = (Ns[k] - x[k] * Ns[3]) * iw;
    dv[k] = (Nt[k] - x[k] * Nt[3]) * iw;
  }
}
template <int D>
__device__ __forceinline__ void point_only(const double* __restrict__ cf, double s, double t, double x[3]) {
  double N[4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double* p = cf + c * 25;
    double n = 0.0;
#pragma unroll
    for (int j = D; j >= 0; --j) {
      double r = p[j * 5 + D];
#pragma unroll
      for (int i = D - 1; i >= 0; --i) r = fma(r, s, p[j * 5 + i]);
      n = fma(n, t, r);
    }
    N[c] = n;
  }
  const double iw = 1.0 / N[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) x[k] = N[k] * iw;
}
__device__ __forceinline__ double sqrt_g_of(const double du[3], const double dv[3]) {
  const double n0 = du[1] * dv[2] - du[2] * dv[1];
  const double n1 = du[2] * dv[0] - du[0] * dv[2];
  const double n2 = du[0] * dv[1] - du[1] * dv[0];
  return sqrt(n0 * n0 + n1 * n1 + n2 * n2);
}

// polynomial of degree DEG with coefficients c[0..DEG]
template <int DEG>
__device__ __forceinline__ double horner(const double* c, double s) {
  double r = c[DEG];
#pragma unroll
  for (int k = DEG - 1; k >= 0; --k) r = fma(r, s, c[k]);
  return r;
}
template <int DEG>
__device__ __forceinline__ double horner_d(const double* c, double s) {
  if constexpr (DEG == 0) {
    return 0.0;
  } else {
    double r = DEG * c[DEG];
#pragma unroll
    for (int k = DEG - 1; k >= 1; --k) r = fma(r, s, k * c[k]);
    return r;
  }
}

// shape data of one point: NC channels x NL values (real).
// scalar: value; Maxwell: field x/y/z and surface divergence
// (spaces.cpp:257-307).  tab: element tables in smem.
template <class KT>
__device__ __forceinline__ void shapes(const double* __restrict__ tab, double s, double t, double h,
                                       const double du[3], const double dv[3], double sg,
                                       double out[KT::NC][KT::NL]) {
  if constexpr (KT::KIND != 2) {
    constexpr int Q = KT::Q;
    double bu[Q + 1], bv[Q + 1];
#pragma unroll
    for (int i = 0; i <= Q; ++i) {
      bu[i] = horner<Q>(tab + i * (Q + 1), s);
      bv[i] = horner<Q>(tab + (Q + 1) * (Q + 1) + i * (Q + 1), t);
    }
#pragma unroll
    for (int j = 0; j <= Q; ++j)
#pragma unroll
      for (int i = 0; i <= Q; ++i) out[0][i + (Q + 1) * j] = bu[i] * bv[j];
  } else {
    constexpr int P = KT::Q;
    const double* tpu = tab;
    const double* tpv = tab + (P + 1) * (P + 1);
    const double* tqu = tab + 2 * (P + 1) * (P + 1);
    const double* tqv = tqu + P * P;
    double bpu[P + 1], bpv[P + 1], dpu[P + 1], dpv[P + 1], bqu[P], bqv[P];
    const double ih = 1.0 / h;
#pragma unroll
    for (int i = 0; i <= P; ++i) {
      bpu[i] = horner<P>(tpu + i * (P + 1), s);
      bpv[i] = horner<P>(tpv + i * (P + 1), t);
      dpu[i] = horner_d<P>(tpu + i * (P + 1), s) * ih;
      dpv[i] = horner_d<P>(tpv + i * (P + 1), t) * ih;
    }
#pragma unroll
    for (int i = 0; i < P; ++i) {
      bqu[i] = horner<P - 1>(tqu + i * P, s);
      bqv[i] = horner<P - 1>(tqv + i * P, t);
    }
    const double ig = 1.0 / sg;
    int l = 0;
#pragma unroll
    for (int j = 0; j < P; ++j)
#pragma unroll
      for (int i = 0; i <= P; ++i, ++l) {
        const double b = bpu[i] * bqv[j];
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k][l] = ig * du[k] * b;
        out[3][l] = ig * dpu[i] * bqv[j];
      }
#pragma unroll
    for (int j = 0; j <= P; ++j)
#pragma unroll
      for (int i = 0; i < P; ++i, ++l) {
        const double b = bqu[i] * bpv[j];
#pragma unroll
        for (int k = 0; k < 3; ++k) out[k][l] = ig * dv[k] * b;
        out[3][l] = ig * bqu[i] * dpv[j];
      }
  }
}

// element tables (u, v) for grid position (ix, iy) into smem
template <class KT>
__device__ __forceinline__ void load_tables(double* dst, const double* __restrict__ ta,
                                            const double* __restrict__ tb, int ix, int iy, int tid,
                                            int nthreads) {
  if constexpr (KT::KIND != 2) {
    constexpr int T = (KT::Q + 1) * (KT::Q + 1);
    for (int i = tid; i < 2 * T; i += nthreads) dst[i] = (i < T) ? ta[ix * T + i] : ta[iy * T + i - T];
  } else {
    constexpr int P = KT::Q, TP = (P + 1) * (P + 1), TQ = P * P;
    for (int i = tid; i < 2 * TP + 2 * TQ; i += nthreads) {
      double v;
      if (i < TP) v = ta[ix * TP + i];
      else if (i < 2 * TP) v = ta[iy * TP + i - TP];
      else if (i < 2 * TP + TQ) v = tb[ix * TQ + i - 2 * TP];
      else v = tb[iy * TQ + i - 2 * TP - TQ];
      dst[i] = v;
    }
  }
}

}  // namespace dev
}  // namespace igb
