// Device-resident H² operator (assembly + matvec on one B200).
#pragma once

#include <cuda_runtime.h>

#include <chrono>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "igb_host.hpp"

namespace igb {

struct AssemblyTimes {  // milliseconds, CUDA events on the assembly stream
  double plan_host = 0, upload = 0, elements = 0, images = 0, couplings = 0, regular = 0,
         singular[4] = {0, 0, 0, 0}, total_device = 0, total_wall = 0, scatter = 0;
};

struct DeviceBytes {
  size_t near = 0, far = 0, moments = 0, other = 0;
};

class H2Device {
 public:
  // flags bit1 (IGB_H2_STORED_COUPLINGS): store the far couplings (reference
  // format) instead of evaluating them inside the matvec; bit3
  // (IGB_H2_FUSED_COUPLINGS): always evaluate them; neither: chosen per kind
  // and size after the block partition
  // world > 1: this rank assembles and applies the block rows of its level-1
  // clusters (build_local_plan); apply via dist_phase1 / all-gather /
  // dist_phase2 / all-reduce
  H2Device(std::shared_ptr<const Discretization> d, int m, double eta, int far_order,
           int sing_order, int device, int flags = 0, int world = 1, int rank = 0);
  ~H2Device();
  H2Device(const H2Device&) = delete;
  H2Device& operator=(const H2Device&) = delete;

  const Discretization& disc() const { return *disc_; }
  enum { kStoredCouplings = 2, kDevicePartition = 4, kFusedCouplings = 8 };  // include/igabem_b200.h flags
  bool stored_couplings() const { return (flags_ & kStoredCouplings) != 0; }
  const H2Plan& plan() const { return plan_; }
  const LocalPlan& local_plan() const { return lp_; }
  // multi-GPU matvec: phase 1 (x -> packed owned up moments, `send` holds
  // send_count() scalars), caller all-gathers into `recv` (world * send_count),
  // phase 2 (recv -> partial y over all DOFs), caller all-reduces y
  size_t send_count() const { return static_cast<size_t>(lp_.pack_max) * nch_ * plan_.m * plan_.m; }
  void dist_phase1(const double* x, double* send, cudaStream_t s);
  void dist_phase2(const double* recv, double* y, cudaStream_t s);
  bool is_complex() const { return disc_->is_complex(); }
  int dim() const { return disc_->dof_count(); }
  int nch() const { return nch_; }
  int m() const { return plan_.m; }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  const AssemblyTimes& times() const { return times_; }
  DeviceBytes bytes() const { return bytes_; }

  // y = H x.  Scalars are double or interleaved complex<double>.
  void apply_host(const double* x, double* y);
  void apply_device(const double* x, double* y, cudaStream_t s);
  // launches of the matvec graph without copies (benchmarking): x/y are the
  // internal buffers
  double* x_buffer() { return dx_; }
  double* y_buffer() { return dy_; }
  void launch_apply_graph(cudaStream_t s);
  // re-run the device assembly kernels on the resident inputs; returns device ms
  double reassemble();
  // per-phase matvec time (ms summed over iters): coef, leaf_up, upward,
  // zero, far, downward, near_leaf, scatter
  void profile_apply(int iters, double* phase_ms);
  // the level-split matvec graph's kernels launched one after another on the
  // handle's stream, each timed with CUDA events: (name, ms summed over iters)
  std::vector<std::pair<std::string, double>> profile_kernels(int iters);
  // matvec phases 1-4 on host x (through the far field and its slot sums):
  // up and down ([node][c*m^2 + nu], Scalar) to host
  void far_field(const double* x, double* up_out, double* down_out);
  // unordered far pairs the symmetric far kernels evaluate: [leaf level, above]
  long long sym_pairs(int which) const { return sym_pairs_[which]; }
  // leaf-level far pairs applied as stored element blocks (LeafBlocks) and their bytes
  long long leaf_block_pairs() const { return n_leaf_blocks_; }
  size_t leaf_block_bytes() const { return leaf_block_bytes_; }
  // bytes of block rows one matvec streams (near field + leaf blocks as the leaf kernel reads them)
  size_t block_stream_bytes() const {
    const size_t nl2 = static_cast<size_t>(disc_->local_count()) * disc_->local_count() * (is_complex() ? 16 : 8);
    return lb_sym_near_ ? static_cast<size_t>(n_lb_total_) * nl2 : bytes_.near + leaf_block_bytes_;
  }
  // `steps` x (device assembly + `matvecs` matvecs), CUDA events; returns ms
  double bench_steps(int steps, int matvecs, double* assembly_ms);
  int assembly_kernel_launches() const { return assembly_kernels_; }
  size_t upload_bytes() const { return upload_bytes_; }
  int apply_kernel_launches() const { return apply_launches_; }

  // introspection (host copies, reference layouts)
  void near_blocks(long long first, long long count, double* out) const;  // [q][la][lb]
  void couplings(long long first, long long count, double* out) const;    // [q][mu][nu] (col-major K)
  void moments(double* out) const;                                        // [e][l][row] real
  void images(double* out) const;                                         // [node][nu][3]

 private:
  template <class KT> void assemble_impl(std::chrono::steady_clock::time_point t_wall0);
  template <class KT> void stage_elements();
  template <class KT> void stage_plan();
  template <class KT> void launch_element_phase(cudaEvent_t* ev, int& launched);
  template <class KT> void launch_plan_phase(cudaEvent_t* ev, int& launched);
  template <class KT> void run_assembly();
  void collect_times(cudaEvent_t* ev);
  // assembly events
  enum { kEvStart, kEvElements, kEvCoincident, kEvEdge, kEvVertex, kEvUploaded, kEvPlanPhase, kEvImages,
         kEvCouplings, kEvRegular, kEvScatter, kAsmEvents };
  template <class KT> void enqueue_apply(const double* x, double* y, cudaStream_t s, cudaEvent_t* pev);
  using KernelMarks = std::vector<std::pair<const char*, cudaEvent_t>>;
  template <class KT> void enqueue_apply_split(const double* x, double* y, cudaStream_t s, KernelMarks* prof = nullptr);
  // the single-GPU symmetric far field is captured as the level-split graph
  bool split_graph() const { return sym_far_ && lp_.world == 1 && plan_.depth >= 1; }
  template <class KT> void enqueue_phase1(const double* x, double* send, cudaStream_t s, cudaEvent_t* pev, int& n);
  template <class KT> void enqueue_phase2(const double* recv, double* y, cudaStream_t s, cudaEvent_t* pev, int& n);
  template <class F> void dispatch_kind(F&& f);
  void enqueue_apply_dispatch(const double* x, double* y, cudaStream_t s, cudaEvent_t* pev);

  std::shared_ptr<const Discretization> disc_;
  H2Plan plan_;
  LocalPlan lp_;
  int device_ = 0, nch_ = 1, flags_ = 0;
  struct Opts {
    int m;
    double eta;
    int far_order, sing_order, world, rank;
  } opt_{};
  int nfar_ = 0, nsing_ = 0;
  SingList sing_items_[4];          // singular items from the mesh topology (stage 1)
  double* d_sing_blk_[4] = {};      // their blocks [item][la][lb], Scalar
  cudaStream_t stream_ = nullptr;
  cudaStream_t aux_ = nullptr;      // stage-2 uploads (overlap the stage-1 kernels)
  cudaStream_t up_stream_ = nullptr;
  AssemblyTimes times_;
  DeviceBytes bytes_;

  // device arrays (raw allocations, owned)
  std::vector<void*> allocs_;
  template <class T> T* dalloc(size_t n);  // stream-ordered, from the per-device pool
  void release_memory();
  template <class T> T* upload(const std::vector<T>& v);

  // geometry / space
  double* d_cells_ = nullptr;       // [cell][100] coefficients + [cell][2] origins
  int* d_el_cell_ = nullptr;        // [e]
  int* d_patch_info_ = nullptr;     // per patch: cell_base, pu, pv, nku, nkv, ku_off, kv_off
  double* d_knots_ = nullptr;
  double* d_tab_a_ = nullptr;       // scalar: tab_s; Maxwell: tab_p
  double* d_tab_b_ = nullptr;       // Maxwell: tab_q
  int* d_l2g_ = nullptr;
  double* d_lsign_ = nullptr;
  // plan
  int *d_near_a_ = nullptr, *d_near_b_ = nullptr, *d_near_rs_ = nullptr;
  int *d_far_b_ = nullptr, *d_far_rs_ = nullptr, *d_far_targets_ = nullptr;
  int n_far_targets_ = 0;
  bool sym_far_ = false;  // Laplace m <= 6: lane-tile symmetric far kernel
  bool sym_w_ = false;    // other kinds / m, one GPU: warp-row symmetric far kernel
  bool far_col_ = false;  // Laplace m <= 5, one GPU: column-stream far kernel (k_far_col)
  bool far_only_ = false;  // far_field(): enqueue only phases 1-4
  int n_sym_targets_ = 0;
  int *d_sym_targets_ = nullptr, *d_upper_start_ = nullptr, *d_trans_ = nullptr;
  int *d_col_rs_ = nullptr, *d_col_q_ = nullptr;  // multi-GPU ranks: per-target pair lists (k_far_col_list)
  int n_sym_fine_ = 0, n_sym_coarse_ = 0;  // leaf-level / coarser symmetric targets
  long long sym_pairs_[2] = {0, 0};        // unordered far pairs evaluated by them
  int *d_sym_fine_ = nullptr, *d_sym_coarse_ = nullptr, *d_sym_all_ = nullptr;
  int n_near_rest_ = -1;  // fused leaf far field + near rows: elements without leaf targets (-1: off)
  int* d_near_rest_ = nullptr;
  double* d_slot_ = nullptr;
  // leaf blocks (fused leaf kernel): blocked unordered leaf pairs in CSR by the
  // lower element, their nodes (assembly), the incoming lists of the upper
  // elements, blocks in the block-row layout, transposed products
  long long n_leaf_blocks_ = 0;
  size_t leaf_block_bytes_ = 0;
  int n_lb_total_ = 0;        // block-row positions: blocked far pairs (+ near pairs f >= e when lb_sym_near_)
  bool lb_sym_near_ = false;  // k_leaf_ws: the near field is part of the block rows (stored once per unordered pair)
  int* d_lb_nq_ = nullptr;
  // Helmholtz (one GPU): every leaf-level far pair as a complex element block in rows added
  // to the near rows (k_leaf_blocks_c / k_block_rows_acc); the far kernel keeps the coarse levels
  bool cblk_ = false;
  int n_far_coarse_ = 0;
  int* d_far_coarse_ = nullptr;  // stored couplings + blocks: the far targets above the leaf level
  int *d_cb_rs_ = nullptr, *d_cb_eb_ = nullptr;
  double* d_cb_blk_ = nullptr;
  int *d_low_rs_ = nullptr, *d_low_q_ = nullptr;  // per node: the lower pairs whose slots are written
  int *d_upper_end_ = nullptr, *d_lb_rs_ = nullptr, *d_lb_eb_ = nullptr, *d_lb_ns_ = nullptr;
  int *d_lb_in_rs_ = nullptr, *d_lb_in_k_ = nullptr;
  double *d_lb_blk_ = nullptr, *d_lb_tslot_ = nullptr;
  int *d_far_a_ = nullptr;
  int *d_dof_start_ = nullptr, *d_dof_inc_ = nullptr;
  int *d_near_ea_ = nullptr, *d_el_ = nullptr, *d_pack_nodes_ = nullptr, *d_unpack_nodes_ = nullptr;
  unsigned char* d_owned_ = nullptr;
  double *d_loc_sign_ = nullptr, *d_send_ = nullptr, *d_recv_ = nullptr;
  double *d_tl_ = nullptr, *d_tr_ = nullptr;
  // operator data
  double* d_near_ = nullptr;   // block rows per test element (tiled layout, row_tile_off), Scalar
  double* d_far_ = nullptr;    // [q][mu][nu], Scalar
  double* d_mom_ = nullptr;    // [e][l][row], real
  double* d_img_ = nullptr;    // [node][nu][3]
  double* d_cpts_ = nullptr;   // element caches (assembly scratch)
  double* d_cval_ = nullptr;
  // matvec scratch (Scalar)
  double *dx_ = nullptr, *dy_ = nullptr, *d_coef_ = nullptr, *d_up_ = nullptr, *d_down_ = nullptr,
         *d_loc_ = nullptr;
  double *h_x_pinned_ = nullptr, *h_y_pinned_ = nullptr;
  double* d_nrows_ = nullptr;
  cudaStream_t side_ = nullptr, side2_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr, ev_fork2_ = nullptr, ev_join2_ = nullptr;
  cudaEvent_t ev_apply_done_ = nullptr;  // last apply's final copy (dx_/dy_ hand-off between streams)
  cudaGraphExec_t graph_exec_ = nullptr;
  cudaGraphExec_t graph1_ = nullptr, graph2_ = nullptr;  // multi-GPU phases
  bool near_in_phase2_ = false;  // set while capturing the phase graphs
  int apply_launches_ = 0, phase1_launches_ = 0;
  int assembly_kernels_ = 0, assembly_launches_count_ = 0;
  size_t upload_bytes_ = 0;
  double alloc_ms_ = 0;
  struct AsmState {
    double *gxf = nullptr, *gwf = nullptr, *gxs = nullptr, *gws = nullptr, *lag = nullptr, *cheb = nullptr;
    int *reg = nullptr, *reg_ba = nullptr, *node_patch = nullptr, *node_level = nullptr, *node_sx = nullptr, *node_sy = nullptr;
    int* sing[4][4] = {};
    unsigned char* singm[4][2] = {};
    double kp[4] = {0, 0, 0, 0};
  } as_;
};

// return the memory of destroyed operators (kept reserved for re-use) to the driver
void release_device_memory(int device);

// Dense Galerkin matrix (assembly.cpp:16-53) on one device; `out`: host,
// column-major dof_count^2 Scalar (interleaved complex for Helmholtz/Maxwell)
void dense_assemble(const Discretization& d, int far_order, int sing_order, int device, double* out);

}  // namespace igb
