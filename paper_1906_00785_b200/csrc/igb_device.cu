// Host driver of the device-resident H² single-layer / EFIE operator on one
// B200 (H2Device): the pipelined constructor (singular items from the mesh
// topology first, the block partition behind them), the assembly launches,
// the matvec as CUDA graphs (level-split on one GPU, two phases per rank of the
// row-cluster partition), measurement hooks, introspection and the dense
// Galerkin assembly.  Kernels: igb_kernels_assembly.cuh, igb_kernels_matvec.cuh.
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
#include "igb_kernels_assembly.cuh"
#include "igb_kernels_matvec.cuh"

namespace igb {

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

// device memory an operator can still take: what the driver reports free plus
// what the per-device pool holds but does not use (memory of destroyed
// operators stays reserved there)
static size_t available_device_bytes(int device) {
  size_t free_b = 0, total_b = 0;
  IGB_CUDA(cudaMemGetInfo(&free_b, &total_b));
  uint64_t reserved = 0, used = 0;
  cudaMemPool_t pool = device_pool(device);
  IGB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReservedMemCurrent, &reserved));
  IGB_CUDA(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrUsedMemCurrent, &used));
  return free_b + static_cast<size_t>(reserved > used ? reserved - used : 0);
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

// default fraction of each leaf target's upper far pairs applied as stored
// element blocks (IGB_H2_LEAF_BLOCKS overrides): warp-specialised kernel (c5
// matvec 10.02 / 9.77 / 9.57 / 9.53 ms at 0.5 / 0.6 / 0.7 / 0.8; 10.88 ms before)
// and the one-warp-per-target fused kernel (c5 leaf kernel 7.30 -> 6.71 ms at 0.4)
constexpr double kLeafBlockFractionWs = 0.9, kLeafBlockFraction = 0.4;
// IGB_H2_LEAF_WS=0: the one-warp-per-target fused leaf kernel instead of k_leaf_ws
static bool leaf_ws_enabled() {
  const char* e = getenv("IGB_H2_LEAF_WS");
  return e == nullptr || atoi(e) != 0;
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
  // the setup (boxes, traversal, sort, classes) runs on the device unless the host
  // is asked for (flag 16 / IGB_H2_HOST_PARTITION) or a patch degree exceeds the
  // device kernels' bound; both give bit-identical plans
  bool dev_setup = !(flags_ & 16) && getenv("IGB_H2_HOST_PARTITION") == nullptr;
  for (int p = 0; p < d.geometry().patch_count() && !(flags_ & 4); ++p)
    if (d.geometry().patch(p).kv_u.degree > 15 || d.geometry().patch(p).kv_v.degree > 15) dev_setup = false;
  plan_ = build_plan(d, opt_.m, opt_.eta, opt_.far_order, opt_.sing_order, ((flags_ & 4) || dev_setup) ? device_ : -1);
  lp_ = build_local_plan(d, plan_, opt_.world, opt_.rank);
  times_.plan_host = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  lap("plan");
  // couplings stored or evaluated in every matvec: unless forced, complex kinds
  // store them when they fit in half the free device memory -- their m^4
  // complex kernel evaluations per pair cost more than streaming the block
  // (c4: 6.2 ms per matvec stored at 93 % of HBM vs 14.6 ms evaluated); Laplace
  // always evaluates them (c5: the symmetric FP64 kernel beats the 161 GB stream)
  // (either way the leaf level of the complex kinds is applied as element blocks,
  // k_leaf_blocks_c, and only the coarse levels stream / evaluate couplings)
  if (!(flags_ & (kStoredCouplings | kFusedCouplings)) && opt_.world == 1 && d.is_complex()) {
    const size_t free_b = available_device_bytes(device_);
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
    // complex kinds: all leaf-level far pairs as complex element blocks (ordered rows)
    auto setup_cblk = [&]() {
      {
        double frac = 1.0;
        if (const char* env = getenv("IGB_H2_LEAF_BLOCKS")) frac = atof(env);
        const int ne = d.element_count(), epp = d.elements_per_patch(), leaf_off = P.level_offset[P.depth];
        std::vector<int> cb_rs(ne + 1, 0);
        for (int e = 0; e < ne; ++e) {
          const int t = (e / epp) * P.npp + leaf_off + e % epp;
          cb_rs[e + 1] = cb_rs[e] + (P.far_row_start[t + 1] - P.far_row_start[t]);
        }
        const double need = static_cast<double>(cb_rs[ne]) * NL * NL * 16.0;
        if (frac > 0.0 && cb_rs[ne] > 0 && need <= 0.25 * static_cast<double>(available_device_bytes(device_))) {
          std::vector<int> eb(cb_rs[ne]);
#pragma omp parallel for schedule(static)
          for (int e = 0; e < ne; ++e) {
            const int t = (e / epp) * P.npp + leaf_off + e % epp;
            for (int q = P.far_row_start[t], k = cb_rs[e]; q < P.far_row_start[t + 1]; ++q, ++k) {
              const int sq = P.far_b[q];
              eb[k] = (sq / P.npp) * epp + (sq % P.npp - leaf_off);
            }
          }
          d_cb_rs_ = upload(cb_rs);
          d_cb_eb_ = upload(eb);
          d_cb_blk_ = dalloc<double>(static_cast<size_t>(cb_rs[ne]) * NL * NL * 2);
          cblk_ = true;
          n_leaf_blocks_ = cb_rs[ne] / 2;
          leaf_block_bytes_ = static_cast<size_t>(cb_rs[ne]) * NL * NL * 16;
          sym_pairs_[0] = 0;
        }
      }
    };
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
      {  // k_leaf_ws takes every target: the coarse levels first
        std::vector<int> all(coarse);
        all.insert(all.end(), fine.begin(), fine.end());
        d_sym_all_ = upload(all);
      }
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
        // Leaf blocks: the fused leaf kernel is FP64-bound and leaves HBM idle, so
        // a fraction of every leaf target's upper pairs (the last ones of its
        // row) is applied as stored element blocks M_t K M_s^T instead of being
        // evaluated (k_leaf_blocks; streamed once per unordered pair for both
        // directions).  IGB_H2_LEAF_BLOCKS: the fraction (0 disables).
        double frac = (NL == 16 && leaf_ws_enabled()) ? kLeafBlockFractionWs : kLeafBlockFraction;
        if (const char* env = getenv("IGB_H2_LEAF_BLOCKS")) frac = atof(env);
        frac = std::min(1.0, std::max(0.0, frac));
        const int ne = d.element_count(), leaf_off = P.level_offset[P.depth];
        auto leaf_of = [&](int e) { return (e / epp) * P.npp + leaf_off + e % epp; };
        // warp-specialised kernel: the near field joins the block rows, stored once
        // per unordered pair as well -- row e = [near blocks (e, f), f >= e, the
        // diagonal block halved][blocked far pairs]; k_pack_sym_near copies them from
        // the near storage -- so its stream warps move half the near bytes
        const bool sym_near = NL == 16 && leaf_ws_enabled() && (m == 4 || m == 5) && frac > 0.0;
        const auto t_lb = std::chrono::steady_clock::now();
        auto lb_lap = [&](const char* what) {
          if (getenv("IGB_VERBOSE"))
            fprintf(stderr, "[igb ctor] leaf blocks: %-12s %8.2f ms\n", what,
                    std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_lb).count());
        };
        std::vector<int> lb_rs(ne + 1, 0), upper_end(P.far_row_start.begin() + 1, P.far_row_start.end());
        std::vector<int> n_sym(ne, 0), n_far(ne, 0);
        for (int e = 0; e < ne && sym_near; ++e) {
          const auto first = P.near_b.begin() + P.near_row_start[e], last = P.near_b.begin() + P.near_row_start[e + 1];
          n_sym[e] = static_cast<int>(last - std::lower_bound(first, last, e));
        }
        long long n_far_total = 0;
        for (; frac > 0.0; frac *= 0.5) {  // within a quarter of the free device memory
          n_far_total = 0;
          for (int e = 0; e < ne; ++e) {
            const int t = leaf_of(e), nup = P.far_row_start[t + 1] - P.far_upper_start[t];
            n_far[e] = std::min(nup, static_cast<int>(frac * nup + 0.5));
            n_far_total += n_far[e];
            lb_rs[e + 1] = lb_rs[e] + n_sym[e] + n_far[e];
          }
          const size_t free_b = available_device_bytes(device_);
          const size_t fixed = (static_cast<size_t>(Lp.near_row.size()) * NL * NL + P.far_a.size() * mm) * 8;
          if (static_cast<double>(lb_rs[ne]) * NL * NL * 8 <= 0.25 * (static_cast<double>(free_b) - fixed)) break;
        }
        lb_lap("counts");
        if (frac > 0.0 && n_far_total > 0) {
          const int nb = lb_rs[ne];
          // per position: source element, far node (-1: near block), near slot (-1: far pair)
          std::vector<int> ns(nb, -1), eb(nb), nq(nb, -1), in_rs(ne + 1, 0), in_k(nb);
#pragma omp parallel for schedule(static)
          for (int e = 0; e < ne; ++e) {
            const int t = leaf_of(e);
            int k = lb_rs[e];
            for (int q = P.near_row_start[e + 1] - n_sym[e]; q < P.near_row_start[e + 1]; ++q, ++k) {
              eb[k] = P.near_b[q];
              nq[k] = q;
            }
            upper_end[t] -= n_far[e];
            for (int j = 0; j < n_far[e]; ++j, ++k) {
              const int sq = P.far_b[upper_end[t] + j];
              ns[k] = sq;
              eb[k] = (sq / P.npp) * epp + (sq % P.npp - leaf_off);
            }
          }
          lb_lap("positions");
          for (int k = 0; k < nb; ++k) ++in_rs[eb[k] + 1];
          for (int e = 0; e < ne; ++e) in_rs[e + 1] += in_rs[e];
          {
            std::vector<int> fill(in_rs.begin(), in_rs.end() - 1);
            for (int k = 0; k < nb; ++k) in_k[fill[eb[k]]++] = k;  // ascending k: fixed summation order
          }
          lb_lap("in lists");
          n_leaf_blocks_ = n_far_total;
          leaf_block_bytes_ = static_cast<size_t>(n_far_total) * NL * NL * 8;
          n_lb_total_ = nb;
          lb_sym_near_ = sym_near;
          sym_pairs_[0] -= n_far_total;
          {  // slots the far kernels write: per row s the pairs (s, t), t < s, that t evaluates
            std::vector<int> low_rs(P.n_nodes + 1, 0);
#pragma omp parallel for schedule(static)
            for (int sn = 0; sn < P.n_nodes; ++sn) {
              int c = 0;
              for (int q = P.far_row_start[sn]; q < P.far_upper_start[sn]; ++q)
                c += P.far_trans[q] < upper_end[P.far_b[q]];
              low_rs[sn + 1] = c;
            }
            for (int sn = 0; sn < P.n_nodes; ++sn) low_rs[sn + 1] += low_rs[sn];
            std::vector<int> low_q(low_rs[P.n_nodes]);
#pragma omp parallel for schedule(static)
            for (int sn = 0; sn < P.n_nodes; ++sn) {
              int k = low_rs[sn];
              for (int q = P.far_row_start[sn]; q < P.far_upper_start[sn]; ++q)
                if (P.far_trans[q] < upper_end[P.far_b[q]]) low_q[k++] = q;
            }
            d_low_rs_ = upload(low_rs);
            d_low_q_ = upload(low_q);
          }
          lb_lap("slot lists");
          d_upper_end_ = upload(upper_end);
          d_lb_rs_ = upload(lb_rs);
          d_lb_eb_ = upload(eb);
          d_lb_ns_ = upload(ns);
          if (sym_near) d_lb_nq_ = upload(nq);
          d_lb_in_rs_ = upload(in_rs);
          d_lb_in_k_ = upload(in_k);
          d_lb_blk_ = dalloc<double>(static_cast<size_t>(nb) * NL * NL);
          d_lb_tslot_ = dalloc<double>(static_cast<size_t>(nb) * NL);
          lb_lap("uploads");
        }
      }
      if (sym_w_ && d.is_complex() && ident && P.depth >= 1) setup_cblk();
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
    } else if (stored_couplings() && d.is_complex() && Lp.world == 1 && P.depth >= 2 && mm >= 32 && mm <= 128) {
      // stored couplings streamed for the coarse levels only, the leaf level as element blocks
      bool ident = static_cast<int>(Lp.el.size()) == d.element_count();
      for (size_t i = 0; ident && i < Lp.el.size(); ++i) ident = Lp.el[i] == static_cast<int>(i);
      if (ident) {
        d_upper_start_ = upload(P.far_upper_start);
        d_trans_ = upload(P.far_trans);
        setup_cblk();
        if (cblk_) {
          std::vector<int> coarse;
          for (int t : Lp.far_targets)
            if (P.node_level[t] < P.depth) coarse.push_back(t);
          n_far_coarse_ = static_cast<int>(coarse.size());
          d_far_coarse_ = upload(coarse);
        }
      }
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
  if (n_leaf_blocks_ > 0) {
    if constexpr (KT::KIND == 0 && NL <= 16) {
      auto go = [&](auto kern) {
        kern<<<d.element_count(), 128, 0, stream_>>>(d.element_count(), d_lb_rs_, d_lb_ns_, d.elements_per_patch(), P.npp,
                                                     P.level_offset[P.depth], d_img_, d_mom_, d_lb_blk_);
      };
      if (m == 4) go(k_leaf_blocks<4, NL>);
      else go(k_leaf_blocks<5, NL>);
      ++launched;
      IGB_CUDA(cudaGetLastError());
    }
  }
  if (cblk_) {
    if constexpr (KT::KIND != 0) {
      const size_t smem = (static_cast<size_t>(2 * NL * nch_ * mm + 6 * mm + 1) + 2 * (static_cast<size_t>(mm) * mm + static_cast<size_t>(nch_) * mm * NL)) * 8;
      IGB_CUDA(cudaFuncSetAttribute(k_leaf_blocks_c<KT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
      k_leaf_blocks_c<KT><<<d.element_count(), 128, smem, stream_>>>(
          d.element_count(), m, d_cb_rs_, d_far_rs_, d_far_b_, d_upper_start_, d_trans_, d.elements_per_patch(), P.npp,
          P.level_offset[P.depth], d_img_, d_mom_, g.kp, reinterpret_cast<S*>(d_cb_blk_));
      ++launched;
      IGB_CUDA(cudaGetLastError());
    }
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
  if (lb_sym_near_) {  // the near blocks (e, f), f >= e, into the block rows of k_leaf_ws
    if constexpr (KT::KIND == 0 && NL == 16) {
      k_pack_sym_near<NL><<<grid_for(static_cast<long long>(n_lb_total_) * 32, 128), 128, 0, stream_>>>(
          n_lb_total_, d_lb_nq_, d_lb_eb_, d_lb_rs_, d_near_a_, d_near_rs_, d_near_, d_lb_blk_);
      ++launched;
      IGB_CUDA(cudaGetLastError());
    }
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
    if (cblk_ && !far_only_) {  // + the leaf blocks of the complex kinds
      k_block_rows_acc<S, NL><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, side_>>>(
          nel, d_cb_rs_, d_cb_eb_, reinterpret_cast<const S*>(d_cb_blk_), coef, nrows);
      ++launches;
    }
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
      // leaf blocks: the stored couplings of the coarse levels only
      const bool cbs = cblk_ && !far_only_;
      const int n_ft = cbs ? n_far_coarse_ : n_far_targets_;
      const int* ft = cbs ? d_far_coarse_ : d_far_targets_;
      const unsigned grid = grid_for(static_cast<long long>(std::max(n_ft, 1)) * 32, 256);
      S dw;
      if constexpr (sizeof(S) == 8) {
        dw = 1.0;
      } else {
        const cplx kap = d.kappa();
        const cplx w = d.is_vector() ? -1.0 / (kap * kap) : cplx(1.0, 0.0);
        dw = mk(w.real(), w.imag());
      }
      const S* K = reinterpret_cast<const S*>(d_far_);
      if (n_ft == 0) {
      } else if (mm >= 32) {  // one CTA per target
        const size_t smem = static_cast<size_t>(8) * nch_ * mm * sizeof(S);
        const unsigned nt = static_cast<unsigned>(n_ft);
        if (nch_ == 4) {
          if (mm <= 32) k_far_cta<S, 4, 1><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else if (mm <= 64) k_far_cta<S, 4, 2><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else k_far_cta<S, 4, 4><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        } else {
          if (mm <= 32) k_far_cta<S, 1, 1><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else if (mm <= 64) k_far_cta<S, 1, 2><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
          else k_far_cta<S, 1, 4><<<nt, 256, smem, s>>>(ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        }
      } else if (nch_ == 4) {
        if (mm <= 32) k_far<S, 4, 1><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else if (mm <= 64) k_far<S, 4, 2><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else k_far<S, 4, 4><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
      } else {
        if (mm <= 32) k_far<S, 1, 1><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else if (mm <= 64) k_far<S, 1, 2><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
        else k_far<S, 1, 4><<<grid, 256, 0, s>>>(n_ft, ft, d_far_rs_, d_far_b_, K, mm, up, dw, down);
      }
    } else if (sym_far_) {
      const unsigned gsym = grid_for(static_cast<long long>(n_sym_targets_) * 32, 256);
      double* dn = reinterpret_cast<double*>(down);
      const double* upd = reinterpret_cast<const double*>(up);
      if (far_col_) {  // one GPU, m <= 5 (graphs without the level split: depth 0)
        switch (m) {
          case 2: k_far_col<2, 4, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_ + 1, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          case 3: k_far_col<3, 4, 1><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_ + 1, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          case 4: k_far_col<4, 3, 2><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_ + 1, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
          default: k_far_col<5, 2, 2><<<gsym, 256, 0, s>>>(n_sym_targets_, d_sym_targets_, d_upper_start_, d_far_rs_ + 1, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_); break;
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
      // leaf blocks (Helmholtz): the leaf level is applied as blocks, the far kernel keeps the rest
      const bool cb = cblk_ && !far_only_;
      const int n_tg = cb ? n_sym_coarse_ : n_sym_targets_;
      const int* tg = cb ? d_sym_coarse_ : d_sym_targets_;
      const unsigned gsym = grid_for(static_cast<long long>(std::max(n_tg, 1)) * 32, 256);
      S* sl = reinterpret_cast<S*>(d_slot_);
      const int R = (mm + 31) / 32;
      const size_t smem = static_cast<size_t>(8) * 32 * R * PW * 8;
      if (R == 1)
        k_far_sym_w<KT, 1><<<gsym, 256, smem, s>>>(n_tg, tg, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else if (R == 2)
        k_far_sym_w<KT, 2><<<gsym, 256, smem, s>>>(n_tg, tg, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else if (R == 3)
        k_far_sym_w<KT, 3><<<gsym, 256, smem, s>>>(n_tg, tg, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      else
        k_far_sym_w<KT, 4><<<gsym, 256, smem, s>>>(n_tg, tg, d_upper_start_, d_far_rs_, d_far_b_,
                                                   d_trans_, d_img_, mm, up, kp, down, sl);
      ++launches;
      const int stride = rows * static_cast<int>(sizeof(S) / 8);
      pdl_launch(k_far_lower<false>, grid_for(static_cast<long long>(P.n_nodes) * stride, 256), 256, 0, s, 
          P.n_nodes, stride, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, reinterpret_cast<double*>(down),
          cb ? 2 : 0, cb ? npp : 1, cb ? P.level_offset[L] : 0);
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
    if (cblk_) {
      k_block_rows_acc<S, NL><<<grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, s>>>(
          nel, d_cb_rs_, d_cb_eb_, reinterpret_cast<const S*>(d_cb_blk_), coef, nrows);
      ++launches;
    }
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
      nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, down, nrows, loc,
      static_cast<const int*>(nullptr), static_cast<const int*>(nullptr), static_cast<const S*>(nullptr));
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
  // warp-specialised leaf kernel (k_leaf_ws): far warps + stream warps per SM
  const bool leaf_ws = fused && leaf_ws_enabled() && NL == 16 && (m == 4 || m == 5);
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
  bool up_w = false;
  if constexpr (KT::KIND == 0 && NL == 16) {
    if (leaf_ws && nel == d.element_count() && rows <= 32) {  // one warp per element, coalesced moments
      up_w = true;
      pdl_launch(k_leaf_up_w<NL>, grid_for(static_cast<long long>(nel) * 32, 256), 256, 0, s, nel, rows, epp, npp,
          P.level_offset[L], static_cast<const double*>(d_mom_), reinterpret_cast<const double*>(x),
          static_cast<const int*>(d_l2g_), static_cast<const double*>(d_lsign_), reinterpret_cast<double*>(up),
          reinterpret_cast<double*>(down), ndown, reinterpret_cast<double*>(coef));
    }
  }
  if (!up_w)
    pdl_launch(k_leaf_up_x<S, NL>, grid_for(std::max(ndown, static_cast<long long>(nel) * rows), 256), 256, 0, s,
        nel, rows, epp, npp, P.level_offset[L], d_mom_, x, d_l2g_, d_lsign_, up, down, ndown,
        static_cast<S*>(leaf_ws ? coef : nullptr));
  ++launches;
  tick("leaf_up");
  if (!prof && !leaf_ws) {
    IGB_CUDA(cudaEventRecord(ev_fork2_, s));
    IGB_CUDA(cudaStreamWaitEvent(side2_, ev_fork2_, 0));
  }
  // leaf blocks: off for the far-field introspection (phase 4 output of all pairs)
  const bool blocks = fused && n_leaf_blocks_ > 0 && !far_only_;
  const int* far_end = d_far_rs_ + 1;
  auto far_sym = [&](cudaStream_t st, int n, const int* targets) {
    if (n == 0) return;
    const unsigned g = grid_for(static_cast<long long>(n) * 32, 256);
    if (far_col_) {  // column stream: m <= 5
#define IGB_FC(M_, MB_, C_) k_far_col<M_, MB_, C_><<<g, 256, 0, st>>>(n, targets, d_upper_start_, far_end, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_)
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
    if (blocks) {  // only the slots the far kernels wrote (the blocked pairs have none)
      pdl_launch(k_far_lower_list, grid_for(static_cast<long long>(P.n_nodes) * mm, 256), 256, 0, st,
          P.n_nodes, mm, static_cast<const int*>(d_low_rs_), static_cast<const int*>(d_low_q_),
          static_cast<const double*>(d_slot_), dn, which, npp, P.level_offset[L]);
      ++launches;
      return;
    }
    pdl_launch(k_far_lower<false>, grid_for(static_cast<long long>(P.n_nodes) * mm, 256), 256, 0, st, 
        P.n_nodes, mm, d_far_rs_, d_upper_start_, d_far_b_, d_owned_, d_slot_, dn, which, npp, P.level_offset[L]);
    ++launches;
  };
  if (leaf_ws) {
    // one stream: upward pass, then k_leaf_ws -- its far warps evaluate the far
    // field of every level (coarse targets first) while its stream warps move the
    // near rows and leaf blocks --, slot sums, downward pass, leaf transform
    if constexpr (KT::KIND == 0 && NL == 16) {
      for (int l = L - 1; l >= 0; --l) {
        const long long tot = (l == 0 ? static_cast<long long>(np) : static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * (l - 1)))) * rows;
        launch_up_level<S>(grid_for(tot, 256), s, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                           d_tl_, d_tr_, up, l == 0 ? 0 : Lp.c0, l == 0 ? 0 : Lp.c1);
        ++launches;
      }
      tick("upward");
      LeafBlocks lbk{far_end, nullptr, nullptr, nullptr, nullptr};
      if (blocks) lbk = LeafBlocks{d_upper_end_, d_lb_rs_, d_lb_eb_, d_lb_blk_, d_lb_tslot_};
      auto ws_launch = [&](auto kern, size_t smem) {
        int nsm = 0;
        IGB_CUDA(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, device_));
        IGB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
        kern<<<nsm, 32 * (ws::kFarWarps + ws::kStreamWarps), smem, s>>>(
            n_sym_coarse_ + n_sym_fine_, d_sym_all_, d.element_count(), d_upper_start_, lbk, d_far_b_, d_trans_, d_img_,
            upd, dn, d_slot_, (blocks && lb_sym_near_) ? nullptr : d_near_rs_, d_near_b_,
            reinterpret_cast<const double*>(d_near_), reinterpret_cast<const double*>(coef),
            reinterpret_cast<double*>(nrows));
      };
      if (m == 4) ws_launch(k_leaf_ws<4, NL, 2>, ws::Layout<4, NL>::BYTES);
      else ws_launch(k_leaf_ws<5, NL, 2>, ws::Layout<5, NL>::BYTES);
      ++launches;
      tick("far_near");
      far_lower(s, 0);
      tick("far_lower");
      if (!prof) IGB_CUDA(cudaStreamWaitEvent(s, ev_join_, 0));
      if (far_only_) return;  // introspection: stop after the far field (phase 4)
      for (int l = 0; l < L; ++l) {
        const long long tot = static_cast<long long>(Lp.c1 - Lp.c0) * (1LL << (2 * l)) * rows;
        launch_down_level<S>(grid_for(tot, 256), s, np, l, npp, P.level_offset[l], P.level_offset[l + 1], m, nch_,
                             d_tl_, d_tr_, down, Lp.c0, Lp.c1);
        ++launches;
      }
      tick("downward");
      pdl_launch(k_leaf_down<S, NL>, grid_for(static_cast<long long>(nel) * NL, 256), 256, 0, s,
          nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, down, nrows, loc,
          static_cast<const int*>(blocks ? d_lb_in_rs_ : nullptr), static_cast<const int*>(blocks ? d_lb_in_k_ : nullptr),
          blocks ? reinterpret_cast<const S*>(d_lb_tslot_) : static_cast<const S*>(nullptr));
      tick("leaf_down");
      pdl_launch(k_scatter<S>, grid_for(d.dof_count(), 256), 256, 0, s, d.dof_count(), d_dof_start_, d_dof_inc_, d_loc_sign_, loc, y);
      launches += 2;
      tick("scatter");
      IGB_CUDA(cudaGetLastError());
      apply_launches_ = launches;
    }
    return;
  }
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
      LeafBlocks lbk{far_end, nullptr, nullptr, nullptr, nullptr};
      if (blocks) lbk = LeafBlocks{d_upper_end_, d_lb_rs_, d_lb_eb_, d_lb_blk_, d_lb_tslot_};
      auto fused_launch = [&](auto kern) {
        kern<<<grid_for(nw * 32, 256), 256, 0, s>>>(
            n_sym_fine_, d_sym_fine_, n_near_rest_, d_near_rest_, epp, npp, P.level_offset[L], d_upper_start_,
            lbk, d_far_b_, d_trans_, d_img_, upd, dn, d_slot_, d_owned_, d_near_rs_, d_near_b_,
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
      nel, d_el_, rows, epp, npp, P.level_offset[L], d_mom_, down, nrows, loc,
      static_cast<const int*>(blocks ? d_lb_in_rs_ : nullptr), static_cast<const int*>(blocks ? d_lb_in_k_ : nullptr),
      blocks ? reinterpret_cast<const S*>(d_lb_tslot_) : static_cast<const S*>(nullptr));
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
  if (n_leaf_blocks_ > 0 && !cblk_)  // Laplace: the blocked pairs' slots were written here; apply() never rewrites them
    IGB_CUDA(cudaMemsetAsync(d_slot_, 0, plan_.far_a.size() * static_cast<size_t>(plan_.m) * plan_.m * sizeof(double), stream_));
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
        const size_t src = static_cast<size_t>(rs - r0) * nl * nl + row_tile_off(cnt * nl, nl, la, static_cast<int>(q - rs) * nl + lb);
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
