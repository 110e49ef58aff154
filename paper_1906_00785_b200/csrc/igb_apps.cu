// SURVEY 8(f) on the B200: the callers of the operator around the hot path.
//   * device-resident restarted GMRES (MGS + one re-orthogonalisation, true
//     residual restarts, best iterate) and CG -- solver.hpp:54-200, same
//     algorithm, vectors never leave HBM, only Hessenberg columns come back;
//   * load vectors b_i = <g, phi_i> (assembly.cpp:55-93) from data values at
//     device-computed quadrature points;
//   * single-layer potentials (operators.cpp:112-208).
// All reductions are fixed-order (deterministic run to run).
#include <chrono>
#include <complex>
#include <cstring>
#include <limits>
#include <vector>

#include "igb_apps.hpp"
#include "igb_common.cuh"

namespace igb {
namespace dev {

// ------------------------------------------------ deterministic BLAS-1
constexpr int kRedBlocks = 296, kRedThreads = 256;

__device__ __forceinline__ double conj_mul(double a, double b) { return a * b; }
__device__ __forceinline__ cd conj_mul(cd a, cd b) { return mk(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x); }

template <class S>
__device__ __forceinline__ S block_reduce(S v, S* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) sh[threadIdx.x] = sh[threadIdx.x] + sh[threadIdx.x + o];
    __syncthreads();
  }
  return sh[0];
}
// partial[b] = sum over the block's grid-stride share of conj(a) * b
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_dot_partial(int n, const S* __restrict__ a, const S* __restrict__ b,
                                                             S* __restrict__ partial) {
  __shared__ S sh[kRedThreads];
  S acc = zero<S>();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    acc = acc + conj_mul(a[i], b[i]);
  const S r = block_reduce(acc, sh);
  if (threadIdx.x == 0) partial[blockIdx.x] = r;
}
template <class S>
__global__ void __launch_bounds__(kRedThreads) k_dot_final(int nb, const S* __restrict__ partial, S* __restrict__ out) {
  __shared__ S sh[kRedThreads];
  S acc = zero<S>();
  for (int i = threadIdx.x; i < nb; i += blockDim.x) acc = acc + partial[i];
  const S r = block_reduce(acc, sh);
  if (threadIdx.x == 0) *out = r;
}
// y += sgn * (*alpha) * x  (alpha on the device)
template <class S>
__global__ void k_axpy_dev(int n, double sgn, const S* __restrict__ alpha, const S* __restrict__ x, S* __restrict__ y) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const S a = *alpha * sgn;
  y[i] = y[i] + a * x[i];
}
template <class S>
__global__ void k_axpby(int n, S a, const S* __restrict__ x, S b, S* __restrict__ y) {  // y = a x + b y
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = a * x[i] + b * y[i];
}
template <class S>
__global__ void k_sub(int n, const S* __restrict__ a, const S* __restrict__ b, S* __restrict__ out) {  // a - b
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = a[i] + b[i] * -1.0;
}
// x += V(:, 0:k) y  (y on the device)
template <class S>
__global__ void k_gemv_update(int n, int k, const S* __restrict__ V, size_t ldv, const S* __restrict__ y,
                              S* __restrict__ x) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  S acc = zero<S>();
  for (int j = 0; j < k; ++j) acc = acc + V[j * ldv + i] * y[j];
  x[i] = x[i] + acc;
}

// ------------------------------------------------------ load vectors
struct SpaceArgs {
  const double* cells;
  const int* el_cell;
  const double* tab_a;
  const double* tab_b;
  int level, epp;
  double h;
};
// quadrature points x(e, q), q = a + n b (assembly.cpp:66-72)
__global__ void k_quad_points(int ne, int n, SpaceArgs g, const double* __restrict__ gx, double* __restrict__ pts) {
  const long long idx = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  const int nq = n * n;
  if (idx >= static_cast<long long>(ne) * nq) return;
  const int e = static_cast<int>(idx / nq), q = static_cast<int>(idx % nq), a = q % n, b = q / n;
  const int n1 = 1 << g.level, r = e % g.epp, ix = r % n1, iy = r / n1;
  const double* cf = g.cells + static_cast<size_t>(g.el_cell[e]) * kCellStride;
  double x[3], du[3], dv[3];
  jet<4>(cf, ix * g.h + g.h * gx[a] - cf[100], iy * g.h + g.h * gx[b] - cf[101], x, du, dv);
  for (int k = 0; k < 3; ++k) pts[idx * 3 + k] = x[k];
}
// per element load vector: scalar kinds b_l = sum_q w g phi_l; Maxwell
// b_l = sum_q w (E . j_l) (bilinear, no conjugation; assembly.cpp:76-84)
template <class KT>
__global__ void __launch_bounds__(128) k_rhs_local(int n, SpaceArgs g, const double* __restrict__ gx,
                                                   const double* __restrict__ gw, const double* __restrict__ gvals,
                                                   double* __restrict__ bloc) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NC = KT::NC;
  __shared__ double cf[104];
  __shared__ double tab[KT::TABN];
  __shared__ S red[128];
  const int e = blockIdx.x, tid = threadIdx.x;
  const int n1 = 1 << g.level, r = e % g.epp, ix = r % n1, iy = r / n1;
  for (int i = tid; i < 104; i += 128) cf[i] = g.cells[static_cast<size_t>(g.el_cell[e]) * kCellStride + i];
  load_tables<KT>(tab, g.tab_a, g.tab_b, ix, iy, tid, 128);
  __syncthreads();
  const int nq = n * n;
  S part[NL];
#pragma unroll
  for (int l = 0; l < NL; ++l) part[l] = zero<S>();
  for (int q = tid; q < nq; q += 128) {
    const int a = q % n, b = q / n;
    double x[3], du[3], dv[3];
    jet<4>(cf, ix * g.h + g.h * gx[a] - cf[100], iy * g.h + g.h * gx[b] - cf[101], x, du, dv);
    const double sg = sqrt_g_of(du, dv);
    const double w = gw[a] * gw[b] * sg * g.h * g.h;
    double sh[NC][NL];
    shapes<KT>(tab, gx[a], gx[b], g.h, du, dv, sg, sh);
    const size_t gi = static_cast<size_t>(e) * nq + q;
    if constexpr (KT::KIND == 2) {
      const cd* E = reinterpret_cast<const cd*>(gvals) + gi * 3;
#pragma unroll
      for (int l = 0; l < NL; ++l) {
        cd s = mk(0.0, 0.0);
        for (int k = 0; k < 3; ++k) s = s + E[k] * sh[k][l];
        part[l] = part[l] + s * w;
      }
    } else {
      const S gv = reinterpret_cast<const S*>(gvals)[gi];
#pragma unroll
      for (int l = 0; l < NL; ++l) part[l] = part[l] + gv * w * sh[0][l];
    }
  }
#pragma unroll
  for (int l = 0; l < NL; ++l) {
    const S v = block_reduce(part[l], red);
    if (tid == 0) reinterpret_cast<S*>(bloc)[static_cast<size_t>(e) * NL + l] = v;
    __syncthreads();
  }
}
template <class S>
__global__ void k_gather(int nd, const int* __restrict__ start, const int* __restrict__ inc,
                         const double* __restrict__ sg, const S* __restrict__ loc, S* __restrict__ out) {
  const int d = blockIdx.x * blockDim.x + threadIdx.x;
  if (d >= nd) return;
  S acc = zero<S>();
  for (int i = start[d]; i < start[d + 1]; ++i) acc = acc + loc[inc[i]] * sg[inc[i]];
  out[d] = acc;
}

// -------------------------------------------------------- potentials
// quadrature nodes: x, w = W sqrt_g h^2 and the density there
// (operators.cpp:26-57,119-126); Maxwell: current j and divergence
template <class KT>
__global__ void __launch_bounds__(128) k_pot_nodes(int n, SpaceArgs g, const double* __restrict__ gx,
                                                   const double* __restrict__ gw, const int* __restrict__ l2g,
                                                   const double* __restrict__ lsign, const double* __restrict__ dens,
                                                   double* __restrict__ nodes) {
  using S = typename KT::S;
  constexpr int NL = KT::NL, NC = KT::NC;
  constexpr int SW = sizeof(S) / 8;
  constexpr int NW = 4 + NC * SW;  // x, y, z, w, density channels
  __shared__ double cf[104];
  __shared__ double tab[KT::TABN];
  const int e = blockIdx.x, tid = threadIdx.x;
  const int n1 = 1 << g.level, r = e % g.epp, ix = r % n1, iy = r / n1;
  for (int i = tid; i < 104; i += 128) cf[i] = g.cells[static_cast<size_t>(g.el_cell[e]) * kCellStride + i];
  load_tables<KT>(tab, g.tab_a, g.tab_b, ix, iy, tid, 128);
  __syncthreads();
  const int nq = n * n;
  const S* d = reinterpret_cast<const S*>(dens);
  for (int q = tid; q < nq; q += 128) {
    const int a = q % n, b = q / n;
    double x[3], du[3], dv[3];
    jet<4>(cf, ix * g.h + g.h * gx[a] - cf[100], iy * g.h + g.h * gx[b] - cf[101], x, du, dv);
    const double sg = sqrt_g_of(du, dv);
    double sh[NC][NL];
    shapes<KT>(tab, gx[a], gx[b], g.h, du, dv, sg, sh);
    double* o = nodes + (static_cast<size_t>(e) * nq + q) * NW;
    o[0] = x[0];
    o[1] = x[1];
    o[2] = x[2];
    o[3] = gw[a] * gw[b] * sg * g.h * g.h;
    S acc[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) acc[c] = zero<S>();
#pragma unroll
    for (int l = 0; l < NL; ++l) {
      const size_t i = static_cast<size_t>(e) * NL + l;
      const S coef = d[l2g[i]] * lsign[i];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = acc[c] + coef * sh[c][l];
    }
#pragma unroll
    for (int c = 0; c < NC; ++c) reinterpret_cast<S*>(o + 4)[c] = acc[c];
  }
}
// u(p) = sum_nodes G(|p - x_n|) rho_n w_n; Maxwell E = SL[j] + k^-2 grad SL[div j]
template <class KT>
__global__ void __launch_bounds__(256) k_pot_eval(long long nn, const double* __restrict__ nodes,
                                                  const double* __restrict__ pts, KParams kp,
                                                  double* __restrict__ out) {
  using S = typename KT::S;
  constexpr int NC = KT::NC;
  constexpr int SW = sizeof(S) / 8;
  constexpr int NW = 4 + NC * SW;
  constexpr int NO = (KT::KIND == 2) ? 3 : 1;
  __shared__ S sh[256];
  const double px = pts[3 * blockIdx.x], py = pts[3 * blockIdx.x + 1], pz = pts[3 * blockIdx.x + 2];
  S acc[NO];
#pragma unroll
  for (int k = 0; k < NO; ++k) acc[k] = zero<S>();
  for (long long i = threadIdx.x; i < nn; i += blockDim.x) {
    const double* o = nodes + i * NW;
    const double d0 = px - o[0], d1 = py - o[1], d2 = pz - o[2];
    const double r2 = d0 * d0 + d1 * d1 + d2 * d2;
    if constexpr (KT::KIND == 0) {
      acc[0] = acc[0] + green(r2, kp, 0.0) * o[4] * o[3];
    } else if constexpr (KT::KIND == 1) {
      const cd rho = reinterpret_cast<const cd*>(o + 4)[0];
      acc[0] = acc[0] + green_c(r2, kp) * rho * o[3];
    } else {
      const cd* jd = reinterpret_cast<const cd*>(o + 4);
      const double r = sqrt(r2);
      const cd gk = green_c(r2, kp);
      // g'(r)/r = g (-i kappa - 1/r) / r  (operators.cpp:198-200)
      const cd mik = mk(kp.ki, -kp.kr);  // -i kappa
      const cd gpr = gk * (mik + mk(-1.0 / r, 0.0)) * (1.0 / r);
      const cd ik2 = mk(-kp.dwx, -kp.dwy);  // 1 / kappa^2
      const cd t = ik2 * gpr * jd[3];
      const double dd[3] = {d0, d1, d2};
#pragma unroll
      for (int k = 0; k < 3; ++k) acc[k] = acc[k] + (gk * jd[k] + t * dd[k]) * o[3];
    }
  }
#pragma unroll
  for (int k = 0; k < NO; ++k) {
    const S v = block_reduce(acc[k], sh);
    if (threadIdx.x == 0) reinterpret_cast<S*>(out)[static_cast<size_t>(blockIdx.x) * NO + k] = v;
    __syncthreads();
  }
}

}  // namespace dev

using namespace dev;

// ================================================================ host side
namespace {
unsigned grid_of(long long n, int bs) { return static_cast<unsigned>((n + bs - 1) / bs); }

struct DevBuf {
  void* p = nullptr;
  DevBuf() = default;
  explicit DevBuf(size_t bytes) { IGB_CUDA(cudaMalloc(&p, bytes ? bytes : 8)); }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};
template <class T>
std::unique_ptr<DevBuf> up_vec(const std::vector<T>& v, cudaStream_t s) {
  auto b = std::make_unique<DevBuf>(v.size() * sizeof(T));
  if (!v.empty()) IGB_CUDA(cudaMemcpyAsync(b->p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
  return b;
}

// device copy of what the load vector / potential kernels need
struct DeviceSpace {
  std::vector<std::unique_ptr<DevBuf>> keep;
  SpaceArgs g{};
  const int *l2g = nullptr, *dof_start = nullptr, *dof_inc = nullptr;
  const double* lsign = nullptr;
  DeviceSpace(const Discretization& d, cudaStream_t s) {
    std::vector<double> cells(d.cells().size() * kCellStride, 0.0);
    for (size_t c = 0; c < d.cells().size(); ++c) {
      const GeomCell& gc = d.cells()[c];
      for (int comp = 0; comp < 4; ++comp)
        for (int j = 0; j <= kMaxGeomDeg; ++j)
          for (int i = 0; i <= kMaxGeomDeg; ++i) cells[c * kCellStride + comp * 25 + j * 5 + i] = gc.coef[comp][j][i];
      cells[c * kCellStride + 100] = gc.u0;
      cells[c * kCellStride + 101] = gc.v0;
    }
    keep.push_back(up_vec(cells, s));
    g.cells = keep.back()->as<double>();
    keep.push_back(up_vec(d.element_cell(), s));
    g.el_cell = keep.back()->as<int>();
    keep.push_back(up_vec(d.is_vector() ? d.tab_p() : d.tab_s(), s));
    g.tab_a = keep.back()->as<double>();
    keep.push_back(up_vec(d.is_vector() ? d.tab_q() : std::vector<double>(1, 0.0), s));
    g.tab_b = keep.back()->as<double>();
    g.level = d.level();
    g.epp = d.elements_per_patch();
    g.h = 1.0 / (1 << d.level());
    keep.push_back(up_vec(d.l2g(), s));
    l2g = keep.back()->as<int>();
    keep.push_back(up_vec(d.lsign(), s));
    lsign = keep.back()->as<double>();
    const int nd = d.dof_count(), nl = d.local_count();
    std::vector<int> start(nd + 1, 0), inc(d.l2g().size());
    for (size_t i = 0; i < d.l2g().size(); ++i) ++start[d.l2g()[i] + 1];
    for (int i = 0; i < nd; ++i) start[i + 1] += start[i];
    std::vector<int> fillp(start.begin(), start.end() - 1);
    for (int e = 0; e < d.element_count(); ++e)
      for (int l = 0; l < nl; ++l) inc[fillp[d.l2g()[static_cast<size_t>(e) * nl + l]]++] = e * nl + l;
    keep.push_back(up_vec(start, s));
    dof_start = keep.back()->as<int>();
    keep.push_back(up_vec(inc, s));
    dof_inc = keep.back()->as<int>();
  }
};

template <class F>
void dispatch(const Discretization& d, F&& f) {
  const int q = d.kind() == kMaxwell ? d.degree() : d.scalar_degree();
  if (d.kind() == kLaplace) {
    switch (q) {
      case 0: f(LapT<0>{}); break;
      case 1: f(LapT<1>{}); break;
      case 2: f(LapT<2>{}); break;
      case 3: f(LapT<3>{}); break;
      case 4: f(LapT<4>{}); break;
      default: throw std::invalid_argument("B200: scalar space degree > 4 not instantiated");
    }
  } else if (d.kind() == kHelmholtz) {
    switch (q) {
      case 0: f(HelmT<0>{}); break;
      case 1: f(HelmT<1>{}); break;
      case 2: f(HelmT<2>{}); break;
      case 3: f(HelmT<3>{}); break;
      case 4: f(HelmT<4>{}); break;
      default: throw std::invalid_argument("B200: scalar space degree > 4 not instantiated");
    }
  } else {
    switch (q) {
      case 1: f(MaxT<1>{}); break;
      case 2: f(MaxT<2>{}); break;
      case 3: f(MaxT<3>{}); break;
      default: throw std::invalid_argument("B200: Maxwell degree > 3 not instantiated");
    }
  }
}

struct StreamGuard {
  cudaStream_t s = nullptr;
  explicit StreamGuard(int device) {
    IGB_CUDA(cudaSetDevice(device));
    IGB_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  }
  ~StreamGuard() {
    if (s) cudaStreamDestroy(s);
  }
};
}  // namespace

int quad_points(const Discretization& d, int quad_order, int device, std::vector<double>& pts) {
  const int n = quad_order > 0 ? quad_order : d.degree() + 2;  // assembly.cpp:60
  std::vector<double> gx, gw;
  gauss_rule(n, gx, gw);
  StreamGuard sg(device);
  DeviceSpace sp(d, sg.s);
  auto dgx = up_vec(gx, sg.s);
  const long long tot = static_cast<long long>(d.element_count()) * n * n;
  DevBuf out(static_cast<size_t>(tot) * 3 * 8);
  k_quad_points<<<grid_of(tot, 256), 256, 0, sg.s>>>(d.element_count(), n, sp.g, dgx->as<double>(), out.as<double>());
  IGB_CUDA(cudaGetLastError());
  pts.resize(static_cast<size_t>(tot) * 3);
  IGB_CUDA(cudaMemcpyAsync(pts.data(), out.p, pts.size() * 8, cudaMemcpyDeviceToHost, sg.s));
  IGB_CUDA(cudaStreamSynchronize(sg.s));
  return n * n;
}

void assemble_rhs(const Discretization& d, int quad_order, int device, const double* gvals, double* b) {
  const int n = quad_order > 0 ? quad_order : d.degree() + 2;
  std::vector<double> gx, gw;
  gauss_rule(n, gx, gw);
  StreamGuard sg(device);
  DeviceSpace sp(d, sg.s);
  auto dgx = up_vec(gx, sg.s);
  auto dgw = up_vec(gw, sg.s);
  const int ne = d.element_count(), nl = d.local_count(), nq = n * n, sw = d.is_complex() ? 2 : 1;
  const size_t nvals = static_cast<size_t>(ne) * nq * (d.is_vector() ? 3 : 1) * sw;
  DevBuf dv(nvals * 8), bloc(static_cast<size_t>(ne) * nl * sw * 8), out(static_cast<size_t>(d.dof_count()) * sw * 8);
  IGB_CUDA(cudaMemcpyAsync(dv.p, gvals, nvals * 8, cudaMemcpyHostToDevice, sg.s));
  dispatch(d, [&](auto kt) {
    using KT = decltype(kt);
    using S = typename KT::S;
    k_rhs_local<KT><<<ne, 128, 0, sg.s>>>(n, sp.g, dgx->as<double>(), dgw->as<double>(), dv.as<double>(),
                                          bloc.as<double>());
    k_gather<S><<<grid_of(d.dof_count(), 256), 256, 0, sg.s>>>(d.dof_count(), sp.dof_start, sp.dof_inc, sp.lsign,
                                                               bloc.as<S>(), out.as<S>());
  });
  IGB_CUDA(cudaGetLastError());
  IGB_CUDA(cudaMemcpyAsync(b, out.p, static_cast<size_t>(d.dof_count()) * sw * 8, cudaMemcpyDeviceToHost, sg.s));
  IGB_CUDA(cudaStreamSynchronize(sg.s));
}

void eval_potential(const Discretization& d, int quad_order, int device, const double* density, int npts,
                    const double* pts, double* out) {
  if (quad_order < 1) throw std::invalid_argument("eval_potential: quadrature order must be positive");
  std::vector<double> gx, gw;
  gauss_rule(quad_order, gx, gw);
  StreamGuard sg(device);
  DeviceSpace sp(d, sg.s);
  auto dgx = up_vec(gx, sg.s);
  auto dgw = up_vec(gw, sg.s);
  const int ne = d.element_count(), nq = quad_order * quad_order, sw = d.is_complex() ? 2 : 1;
  const int nc = d.is_vector() ? 4 : 1, nw = 4 + nc * sw, no = d.is_vector() ? 3 : 1;
  DevBuf dd(static_cast<size_t>(d.dof_count()) * sw * 8), nodes(static_cast<size_t>(ne) * nq * nw * 8),
      dp(static_cast<size_t>(npts) * 3 * 8 + 8), dout(static_cast<size_t>(npts) * no * sw * 8 + 8);
  IGB_CUDA(cudaMemcpyAsync(dd.p, density, static_cast<size_t>(d.dof_count()) * sw * 8, cudaMemcpyHostToDevice, sg.s));
  IGB_CUDA(cudaMemcpyAsync(dp.p, pts, static_cast<size_t>(npts) * 3 * 8, cudaMemcpyHostToDevice, sg.s));
  KParams kp;
  kp.kr = d.kappa().real();
  kp.ki = d.kappa().imag();
  const cplx dw = d.is_vector() ? -1.0 / (d.kappa() * d.kappa()) : cplx(0, 0);
  kp.dwx = dw.real();
  kp.dwy = dw.imag();
  dispatch(d, [&](auto kt) {
    using KT = decltype(kt);
    k_pot_nodes<KT><<<ne, 128, 0, sg.s>>>(quad_order, sp.g, dgx->as<double>(), dgw->as<double>(), sp.l2g, sp.lsign,
                                          dd.as<double>(), nodes.as<double>());
    if (npts > 0)
      k_pot_eval<KT><<<npts, 256, 0, sg.s>>>(static_cast<long long>(ne) * nq, nodes.as<double>(), dp.as<double>(), kp,
                                             dout.as<double>());
  });
  IGB_CUDA(cudaGetLastError());
  IGB_CUDA(cudaMemcpyAsync(out, dout.p, static_cast<size_t>(npts) * no * sw * 8, cudaMemcpyDeviceToHost, sg.s));
  IGB_CUDA(cudaStreamSynchronize(sg.s));
}

// ------------------------------------------------------ Krylov solvers
namespace {
template <class H>  // host scalar: double or std::complex<double>
struct Krylov {
  using D = std::conditional_t<std::is_same_v<H, double>, double, cd>;
  H2Device& A;
  cudaStream_t s;
  int n;
  DevBuf partial, scal;
  explicit Krylov(H2Device& a)
      : A(a), s(a.stream()), n(a.dim()), partial(kRedBlocks * sizeof(D)), scal(4096 * sizeof(D)) {}
  D* sc(int i) const { return scal.as<D>() + i; }
  void dot_dev(const D* a, const D* b, D* out) {
    k_dot_partial<D><<<kRedBlocks, kRedThreads, 0, s>>>(n, a, b, partial.as<D>());
    k_dot_final<D><<<1, kRedThreads, 0, s>>>(kRedBlocks, partial.as<D>(), out);
  }
  H fetch(const D* p) {
    H v;
    IGB_CUDA(cudaMemcpyAsync(&v, p, sizeof(D), cudaMemcpyDeviceToHost, s));
    IGB_CUDA(cudaStreamSynchronize(s));
    return v;
  }
  double norm(const D* a) {
    dot_dev(a, a, sc(4095));
    return std::sqrt(std::real(fetch(sc(4095))));
  }
  static D cvt(H v) {
    if constexpr (std::is_same_v<H, double>)
      return v;
    else
      return mk(v.real(), v.imag());
  }
  void axpby(H a, const D* x, H b, D* y) {
    k_axpby<D><<<grid_of(n, 256), 256, 0, s>>>(n, cvt(a), x, cvt(b), y);
  }
  void apply(const D* x, D* y) { A.apply_device(reinterpret_cast<const double*>(x), reinterpret_cast<double*>(y), s); }
};
template <class T>
T conj_s(const T& v) {
  if constexpr (std::is_same_v<T, double>)
    return v;
  else
    return std::conj(v);
}
}  // namespace

// solver.hpp:54-155 with device vectors
template <class H>
static SolveResult gmres_impl(H2Device& A, const H* b_host, H* x_host, const SolverOpts& o) {
  using D = typename Krylov<H>::D;
  const auto t0 = std::chrono::steady_clock::now();
  Krylov<H> K(A);
  const int n = K.n;
  SolveResult st;
  auto done = [&]() { st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count(); };
  const int kr = std::min(o.restart, n);
  if (kr < 1) throw std::invalid_argument("gmres: restart must be positive");
  if (kr + 2 > 4000) throw std::invalid_argument("gmres: restart too large");
  DevBuf b(n * sizeof(D)), x(n * sizeof(D)), best(n * sizeof(D)), r(n * sizeof(D)), w(n * sizeof(D)),
      V(static_cast<size_t>(n) * (kr + 1) * sizeof(D)), y(kr * sizeof(D));
  IGB_CUDA(cudaMemcpyAsync(b.p, b_host, n * sizeof(D), cudaMemcpyHostToDevice, K.s));
  IGB_CUDA(cudaMemsetAsync(x.p, 0, n * sizeof(D), K.s));
  IGB_CUDA(cudaMemsetAsync(best.p, 0, n * sizeof(D), K.s));
  auto Vc = [&](int j) { return V.as<D>() + static_cast<size_t>(j) * n; };
  const double nb = K.norm(b.as<D>());
  auto finish = [&](const DevBuf& src) {
    IGB_CUDA(cudaMemcpyAsync(x_host, src.p, n * sizeof(D), cudaMemcpyDeviceToHost, K.s));
    IGB_CUDA(cudaStreamSynchronize(K.s));
    done();
    return st;
  };
  if (nb == 0) {
    st.converged = true;
    return finish(x);
  }
  std::vector<H> h(static_cast<size_t>(kr + 1) * kr, H(0)), cs(kr), sn(kr), g(kr + 1);
  auto Hm = [&](int i, int j) -> H& { return h[i + static_cast<size_t>(kr + 1) * j]; };
  double best_res = std::numeric_limits<double>::infinity();
  auto residual = [&]() {  // r = b - A x
    K.apply(x.as<D>(), w.as<D>());
    k_sub<D><<<grid_of(n, 256), 256, 0, K.s>>>(n, b.as<D>(), w.as<D>(), r.as<D>());
    return K.norm(r.as<D>());
  };
  while (st.iterations < o.max_iter) {
    const double nr = residual();
    st.residual = nr / nb;
    if (st.residual < best_res) {
      best_res = st.residual;
      IGB_CUDA(cudaMemcpyAsync(best.p, x.p, n * sizeof(D), cudaMemcpyDeviceToDevice, K.s));
    }
    if (st.residual <= o.tol) {
      st.converged = true;
      return finish(x);
    }
    K.axpby(H(1.0 / nr), r.as<D>(), H(0), Vc(0));
    std::fill(g.begin(), g.end(), H(0));
    g[0] = H(nr);
    int k = 0;
    for (; k < kr && st.iterations < o.max_iter; ++k, ++st.iterations) {
      K.apply(Vc(k), w.as<D>());
      K.dot_dev(w.as<D>(), w.as<D>(), K.sc(kr + 1));  // ||w0||^2
      for (int i = 0; i <= k; ++i) {                  // modified Gram-Schmidt
        K.dot_dev(Vc(i), w.as<D>(), K.sc(i));
        k_axpy_dev<D><<<grid_of(n, 256), 256, 0, K.s>>>(n, -1.0, K.sc(i), Vc(i), w.as<D>());
      }
      K.dot_dev(w.as<D>(), w.as<D>(), K.sc(kr + 2));
      std::vector<H> hc(kr + 3);
      IGB_CUDA(cudaMemcpyAsync(hc.data(), K.scal.p, sizeof(D) * (kr + 3), cudaMemcpyDeviceToHost, K.s));
      IGB_CUDA(cudaStreamSynchronize(K.s));
      const double nw0 = std::sqrt(std::real(hc[kr + 1]));
      double nwr = std::sqrt(std::real(hc[kr + 2]));
      for (int i = 0; i <= k; ++i) Hm(i, k) = hc[i];
      if (nwr < 0.7 * nw0) {  // reorthogonalize once
        for (int i = 0; i <= k; ++i) {
          K.dot_dev(Vc(i), w.as<D>(), K.sc(i));
          k_axpy_dev<D><<<grid_of(n, 256), 256, 0, K.s>>>(n, -1.0, K.sc(i), Vc(i), w.as<D>());
        }
        IGB_CUDA(cudaMemcpyAsync(hc.data(), K.scal.p, sizeof(D) * (k + 1), cudaMemcpyDeviceToHost, K.s));
        IGB_CUDA(cudaStreamSynchronize(K.s));
        for (int i = 0; i <= k; ++i) Hm(i, k) += hc[i];
      }
      const double nw = K.norm(w.as<D>());
      Hm(k + 1, k) = H(nw);
      if (nw > 0) K.axpby(H(1.0 / nw), w.as<D>(), H(0), Vc(k + 1));
      for (int i = 0; i < k; ++i) {  // accumulated Givens rotations
        const H t = cs[i] * Hm(i, k) + sn[i] * Hm(i + 1, k);
        Hm(i + 1, k) = -conj_s(sn[i]) * Hm(i, k) + conj_s(cs[i]) * Hm(i + 1, k);
        Hm(i, k) = t;
      }
      const double rho = std::sqrt(std::norm(Hm(k, k)) + std::norm(Hm(k + 1, k)));
      if (rho == 0) {
        cs[k] = H(1);
        sn[k] = H(0);
      } else {
        cs[k] = conj_s(Hm(k, k)) / H(rho);
        sn[k] = conj_s(Hm(k + 1, k)) / H(rho);
      }
      Hm(k, k) = H(rho);
      Hm(k + 1, k) = H(0);
      const H t = cs[k] * g[k] + sn[k] * g[k + 1];
      g[k + 1] = -conj_s(sn[k]) * g[k] + conj_s(cs[k]) * g[k + 1];
      g[k] = t;
      if (std::abs(g[k + 1]) / nb <= o.tol || nw == 0) {
        ++k;
        ++st.iterations;
        break;
      }
    }
    if (k > 0) {  // upper-triangular solve on the host, x += V y on the device
      std::vector<H> yv(k);
      for (int i = k - 1; i >= 0; --i) {
        H acc = g[i];
        for (int j = i + 1; j < k; ++j) acc -= Hm(i, j) * yv[j];
        yv[i] = acc / Hm(i, i);
      }
      IGB_CUDA(cudaMemcpyAsync(y.p, yv.data(), k * sizeof(D), cudaMemcpyHostToDevice, K.s));
      k_gemv_update<D><<<grid_of(n, 256), 256, 0, K.s>>>(n, k, V.as<D>(), static_cast<size_t>(n), y.as<D>(), x.as<D>());
      IGB_CUDA(cudaStreamSynchronize(K.s));  // yv lifetime
    } else {
      break;
    }
  }
  const double nr = residual();
  st.residual = nr / nb;
  if (st.residual < best_res) {
    best_res = st.residual;
    IGB_CUDA(cudaMemcpyAsync(best.p, x.p, n * sizeof(D), cudaMemcpyDeviceToDevice, K.s));
  }
  st.converged = best_res <= o.tol;
  st.residual = best_res;
  return finish(best);
}

// solver.hpp:159-200 with device vectors
template <class H>
static SolveResult cg_impl(H2Device& A, const H* b_host, H* x_host, const SolverOpts& o) {
  using D = typename Krylov<H>::D;
  const auto t0 = std::chrono::steady_clock::now();
  Krylov<H> K(A);
  const int n = K.n;
  SolveResult st;
  DevBuf x(n * sizeof(D)), r(n * sizeof(D)), p(n * sizeof(D)), ap(n * sizeof(D));
  IGB_CUDA(cudaMemsetAsync(x.p, 0, n * sizeof(D), K.s));
  IGB_CUDA(cudaMemcpyAsync(r.p, b_host, n * sizeof(D), cudaMemcpyHostToDevice, K.s));
  IGB_CUDA(cudaMemcpyAsync(p.p, r.p, n * sizeof(D), cudaMemcpyDeviceToDevice, K.s));
  auto finish = [&]() {
    IGB_CUDA(cudaMemcpyAsync(x_host, x.p, n * sizeof(D), cudaMemcpyDeviceToHost, K.s));
    IGB_CUDA(cudaStreamSynchronize(K.s));
    st.seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return st;
  };
  const double nb = K.norm(r.as<D>());
  if (nb == 0) {
    st.converged = true;
    return finish();
  }
  double rr = nb * nb;
  K.dot_dev(r.as<D>(), r.as<D>(), K.sc(0));
  rr = std::real(K.fetch(K.sc(0)));
  while (st.iterations < o.max_iter) {
    st.residual = std::sqrt(rr) / nb;
    if (st.residual <= o.tol) {
      st.converged = true;
      return finish();
    }
    K.apply(p.as<D>(), ap.as<D>());
    K.dot_dev(p.as<D>(), ap.as<D>(), K.sc(1));
    const double pap = std::real(K.fetch(K.sc(1)));
    if (pap <= 0) break;
    const double alpha = rr / pap;
    K.axpby(H(alpha), p.as<D>(), H(1), x.as<D>());
    K.axpby(H(-alpha), ap.as<D>(), H(1), r.as<D>());
    K.dot_dev(r.as<D>(), r.as<D>(), K.sc(2));
    const double rr_new = std::real(K.fetch(K.sc(2)));
    K.axpby(H(1), r.as<D>(), H(rr_new / rr), p.as<D>());
    rr = rr_new;
    ++st.iterations;
  }
  st.residual = std::sqrt(rr) / nb;
  st.converged = st.residual <= o.tol;
  return finish();
}

SolveResult gmres(H2Device& A, const double* b, double* x, const SolverOpts& o) {
  IGB_CUDA(cudaSetDevice(A.device()));
  if (A.is_complex())
    return gmres_impl<cplx>(A, reinterpret_cast<const cplx*>(b), reinterpret_cast<cplx*>(x), o);
  return gmres_impl<double>(A, b, x, o);
}
SolveResult cg(H2Device& A, const double* b, double* x, const SolverOpts& o) {
  IGB_CUDA(cudaSetDevice(A.device()));
  if (A.is_complex()) return cg_impl<cplx>(A, reinterpret_cast<const cplx*>(b), reinterpret_cast<cplx*>(x), o);
  return cg_impl<double>(A, b, x, o);
}

}  // namespace igb
