/*
 * igabem_b200.h -- C ABI of the B200-native H² boundary-element operator.
 *
 * Drop-in boundary for the reference's hot path (igabem v0.1.0,
 * /root/reference/proj/core): Galerkin assembly and application of the
 * H²-compressed single-layer (Laplace, Helmholtz) and EFIE (Maxwell) operator.
 * Each entry point names the reference interface it replaces.  Plain
 * pointers and sizes only; complex scalars are interleaved (re, im) doubles,
 * i.e. the memory of std::complex<double> / Eigen::VectorXcd.  Every call
 * returns a status code mapping the reference's exception types:
 *   IGB_INVALID_ARGUMENT <- std::invalid_argument   (e.g. h2.cpp:102-110,257)
 *   IGB_LOGIC_ERROR      <- std::logic_error        (e.g. h2.cpp:82,88)
 *   IGB_RUNTIME_ERROR    <- std::runtime_error      (e.g. spaces.cpp:99-104)
 *   IGB_DOMAIN_ERROR     <- std::domain_error       (splines.cpp:62)
 *   IGB_CUDA_ERROR       device failure (no reference analogue)
 * igb_last_error() returns the message of the last failure on this thread.
 */
#ifndef IGABEM_B200_H
#define IGABEM_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  IGB_OK = 0,
  IGB_INVALID_ARGUMENT = 1,
  IGB_LOGIC_ERROR = 2,
  IGB_RUNTIME_ERROR = 3,
  IGB_DOMAIN_ERROR = 4,
  IGB_CUDA_ERROR = 5
};
/* Pde::Kind (pde.hpp:10) */
enum { IGB_LAPLACE = 0, IGB_HELMHOLTZ = 1, IGB_MAXWELL = 2 };
/* PairClass (quadrature.hpp:17) */
enum { IGB_FAR = 0, IGB_VERTEX = 1, IGB_EDGE = 2, IGB_COINCIDENT = 3 };

typedef struct igb_geometry igb_geometry;
typedef struct igb_discretization igb_discretization;
typedef struct igb_h2 igb_h2;

/* PatchSurface (splines.hpp:53-67): clamped knot vectors, homogeneous
 * control points ctrl_w (3 doubles per point, point i + j*count_u) and
 * positive weights. */
typedef struct {
  int degree_u, degree_v;
  int n_knots_u, n_knots_v;
  const double* knots_u;
  const double* knots_v;
  const double* ctrl_w;
  const double* weight;
} igb_patch_desc;

/* Geometry(std::vector<PatchSurface>)  geometry.hpp:40 (topology inference,
 * regularity and orientation checks, geometry.cpp:88-163) */
int igb_geometry_create(int n_patches, const igb_patch_desc* patches, igb_geometry** out);
/* make_sphere(radius, center)  shapes.hpp:21, shapes.cpp:87-205 */
int igb_geometry_sphere(double radius, const double center[3], igb_geometry** out);
/* make_square()  shapes.hpp:16, shapes.cpp:28-30 */
int igb_geometry_square(igb_geometry** out);
/* patch_count(), edge_idents().size(), vertex_idents().size()  geometry.hpp:42-45 */
int igb_geometry_info(const igb_geometry* g, int* n_patches, int* n_edges, int* n_vertices);
void igb_geometry_destroy(igb_geometry* g);

/* Discretization(geometry, Pde{kind, kappa}, degree, rep, level)
 * spaces.hpp:39-40, spaces.cpp:71-115; pde.hpp:19-25 */
int igb_discretization_create(const igb_geometry* g, int kind, double kappa_re, double kappa_im,
                              int degree, int rep, int level, igb_discretization** out);
typedef struct {
  int dof_count, element_count, local_count, level, degree, repetition, kind, patch_count;
} igb_disc_info;
int igb_discretization_info(const igb_discretization* d, igb_disc_info* out);
/* local_to_global / local_sign (spaces.hpp:60-61): element_count*local_count each */
int igb_discretization_l2g(const igb_discretization* d, int* l2g, double* sign);
/* Element (spaces.hpp:15-21): ints[3*e] = patch, ix, iy; dbl[9*e] = h, ox, oy,
 * box min xyz, box max xyz */
int igb_discretization_elements(const igb_discretization* d, int* ints, double* dbl);
/* classify_pair (spaces.hpp:67, spaces.cpp:309-394); maps = swap, flip_u,
 * flip_v of map_a then map_b */
int igb_classify_pair(const igb_discretization* d, int ea, int eb, int* cls, int maps[6]);
void igb_discretization_destroy(igb_discretization* d);

/* H2Options{m, eta, AssemblyOptions{far_order, sing_order}}  h2.hpp:11-15,
 * assembly.hpp:13-20 (0 orders resolve to P+2 / P+3) */
typedef struct {
  int m;
  double eta;
  int far_order;
  int sing_order;
} igb_h2_opts;
/* H2Storage (h2.hpp:49-53), reference convention: entries and bytes of the
 * reference storage format (h2.cpp:380-390) */
typedef struct {
  size_t nearfield_entries, farfield_entries, total_bytes;
} igb_h2_storage;

/* H2Matrix<Scalar>(disc, opts)  h2.hpp:60, h2.cpp:99-129: full assembly on
 * CUDA device `device`.  The discretization may be destroyed afterwards. */
int igb_h2_create(const igb_discretization* d, const igb_h2_opts* opts, int device, igb_h2** out);
/* flags for igb_h2_create_ex: IGB_H2_STORED_COUPLINGS keeps the far couplings
 * in HBM in the reference format (h2.cpp:218-229) and streams them in every
 * matvec; IGB_H2_FUSED_COUPLINGS evaluates them on the fly inside the matvec
 * (same values, no coupling storage).  Neither: Laplace evaluates on the fly,
 * Helmholtz / Maxwell store when the couplings fit in half the free device
 * memory (igb_h2_create always chooses this way). */
/* Setup: igb_h2_create(_ex) builds the element / cluster boxes, the block
 * partition and the pair classes on the device (IGB_H2_DEVICE_PARTITION forces
 * it, IGB_H2_HOST_PARTITION or the environment variable of that name selects
 * the host code; the plans are bit-identical). */
enum { IGB_H2_STORED_COUPLINGS = 2, IGB_H2_DEVICE_PARTITION = 4, IGB_H2_FUSED_COUPLINGS = 8, IGB_H2_HOST_PARTITION = 16 };
int igb_h2_create_ex(const igb_discretization* d, const igb_h2_opts* opts, int device, int flags, igb_h2** out);
/* ---- multi-GPU row-cluster partition ----
 * rank `rank` of `world` assembles and applies the block rows of its level-1
 * clusters.  Matvec: igb_h2_dist_phase1(x -> send), all-gather `send` of
 * every rank into `recv` (rank-major, igb_h2_dist_send_count scalars each),
 * igb_h2_dist_phase2(recv -> y_partial), all-reduce(sum) y_partial.  All
 * pointers are device pointers; work is enqueued on `stream`. */
int igb_h2_create_dist(const igb_discretization* d, const igb_h2_opts* opts, int device, int flags, int world,
                       int rank, igb_h2** out);
int igb_h2_dist_send_count(const igb_h2* h, size_t* scalars);
/* mask[dof] = 1 where this rank's block rows (elements) contribute to y[dof];
 * DOFs set on several ranks are the cut DOFs the y reduction must sum */
int igb_h2_dist_dof_mask(const igb_h2* h, unsigned char* mask);
int igb_h2_dist_phase1(igb_h2* h, const double* x, double* send, void* stream);
int igb_h2_dist_phase2(igb_h2* h, const double* recv, double* y_partial, void* stream);
/* rows()/cols()  h2.hpp:62-63 */
int igb_h2_dim(const igb_h2* h, int* rows);
/* apply(x) / operator*  h2.hpp:64-69, h2.cpp:254-378: host buffers of rows()
 * scalars (double, or interleaved complex for Helmholtz/Maxwell) */
int igb_h2_apply(igb_h2* h, const double* x, double* y);
/* same with device pointers on `stream` (cudaStream_t, NULL = handle stream) */
int igb_h2_apply_device(igb_h2* h, const double* x, double* y, void* stream);
/* storage_report()  h2.hpp:71 */
int igb_h2_storage_report(const igb_h2* h, igb_h2_storage* out);
/* nearfield_pairs().size(), farfield_pairs().size(), tree().node_count() */
int igb_h2_counts(const igb_h2* h, long long* n_near, long long* n_far, int* n_nodes);
/* nearfield_pairs() / farfield_pairs()  h2.hpp:74-75: 2 ints per pair, sorted */
int igb_h2_near_pairs(const igb_h2* h, int* out);
int igb_h2_far_pairs(const igb_h2* h, int* out);
/* tree() (ClusterTree, h2.hpp:25-47): per node patch, level, sx, sy and the
 * box (min xyz, max xyz) */
int igb_h2_tree(const igb_h2* h, int* patch, int* level, int* sx, int* sy, double* boxes);

/* ---- introspection of the assembled operator (parity tests) ---- */
/* near blocks of sorted near pairs [first, first+count): nl*nl scalars each,
 * row-major [la][lb] (= NearBlock::blk, h2.hpp:86-89) */
int igb_h2_near_blocks(const igb_h2* h, long long first, long long count, double* out);
/* couplings of sorted far pairs: m^2*m^2 scalars each, column-major K(nu, mu)
 * (= FarPair::coupling, h2.hpp:90-93) */
int igb_h2_couplings(const igb_h2* h, long long first, long long count, double* out);
/* moments per element: nl x (nch*m^2), [e][l][row], real (= moments_[e]^T,
 * h2.hpp:101) */
int igb_h2_moments(const igb_h2* h, double* out);
/* interpolation-node images per node: m^2 x 3 (h2.cpp:182-196) */
int igb_h2_images(const igb_h2* h, double* out);

/* ---- measurement ---- */
typedef struct {
  double plan_host_ms, upload_ms, elements_ms, images_ms, couplings_ms, regular_ms, coincident_ms,
      edge_ms, vertex_ms, device_total_ms, wall_total_ms,
      scatter_ms; /* singular blocks -> near slots (they are integrated before the partition exists) */
} igb_h2_times;
int igb_h2_assembly_times(const igb_h2* h, igb_h2_times* out);
/* bytes of the device-resident operator in this implementation's format */
int igb_h2_device_bytes(const igb_h2* h, size_t* near, size_t* far, size_t* moments);
/* `iters` back-to-back matvecs on device-resident buffers, CUDA-event timed;
 * *launches = kernels per matvec */
int igb_h2_bench_apply(igb_h2* h, int iters, float* ms, int* launches);
/* re-run the device assembly kernels on the resident inputs (benchmark
 * steps); *device_ms from CUDA events, *launches = kernels launched */
int igb_h2_reassemble(igb_h2* h, double* device_ms, int* launches);
/* per-phase matvec time in ms summed over `iters` (event-separated launches):
 * [coef gather, leaf moments, upward transfer, zero, far couplings, downward
 * transfer, near rows + leaf backward, DOF scatter] (h2.cpp:271-376) */
int igb_h2_profile_apply(igb_h2* h, int iters, double phase_ms[8]);
/* the single-GPU matvec graph's kernels launched one after another, each timed
 * with CUDA events (ms summed over iters); names[k*32 .. k*32+31] = kernel k's
 * role ("far_leaf_near", "upward", ...), *n = kernel count (<= max_n) */
int igb_h2_profile_kernels(igb_h2* h, int iters, int max_n, char* names, double* ms, int* n);
/* unordered far pairs the symmetric far-field kernels evaluate per matvec:
 * pairs[0] on the leaf level, pairs[1] above it (0, 0 for other far kernels) */
int igb_h2_far_work(const igb_h2* h, long long pairs[2]);
/* leaf blocks: leaf-level admissible pairs the matvec applies as stored element
 * blocks M_t K M_s^T (what apply() computes for the pair, h2.cpp:281-290 /
 * 312-326 / 359-371, assembled once) instead of evaluating their couplings:
 * out[0] = unordered pairs, out[1] = bytes of their blocks (0, 0: none),
 * out[2] = bytes of block rows (near field + leaf blocks) one matvec streams --
 * the warp-specialised leaf kernel also stores the near field once per
 * unordered pair.  The environment variable IGB_H2_LEAF_BLOCKS (fraction of
 * every leaf target's pairs, 0 disables) is read at construction. */
int igb_h2_leaf_blocks(const igb_h2* h, long long out[3]);
/* introspection of the far field (phase 4 of H2Matrix::apply, h2.cpp:312-326):
 * runs the matvec on host x through the upward pass and the far field (with
 * the kernel the matvec uses), then copies up and down, each
 * [node][c*m^2 + nu] Scalar (node_count * nch * m^2 scalars); either may be
 * NULL.  Single-GPU handles only. */
int igb_h2_far_field(igb_h2* h, const double* x, double* up, double* down);
/* `steps` x (device assembly + `matvecs` matvecs) on the handle stream,
 * CUDA-event timed; *total_ms, *assembly_ms (sum of assembly device time) */
int igb_h2_bench_steps(igb_h2* h, int steps, int matvecs, double* total_ms, double* assembly_ms);
/* unique (ea <= eb) singular work items per class, indexed by IGB_VERTEX,
 * IGB_EDGE, IGB_COINCIDENT (counts[0] = ordered regular near pairs) */
int igb_h2_class_counts(const igb_h2* h, long long counts[4]);
/* kernels per device assembly and per matvec */
int igb_h2_launch_counts(const igb_h2* h, int* assembly, int* apply);
/* host->device bytes uploaded by igb_h2_create (geometry tables + plan) */
int igb_h2_upload_bytes(const igb_h2* h, size_t* bytes);
void igb_h2_destroy(igb_h2* h);

/* ---- host-only block partition (no device): the cluster tree, dual
 * traversal and pair classification of H2Matrix (h2.cpp:49-97,175-252) ---- */
typedef struct igb_plan igb_plan;
int igb_plan_create(const igb_discretization* d, const igb_h2_opts* opts, igb_plan** out);
/* flags & IGB_H2_DEVICE_PARTITION: the element boxes (spaces.cpp:117-147), the
   cluster boxes and diagonals, the traversal, sort, row starts and transposes of
   the block partition and the classes / maps of the near pairs
   (spaces.cpp:309-394) are computed on CUDA device `device` (
   bit-identical to the host's) */
int igb_plan_create_ex(const igb_discretization* d, const igb_h2_opts* opts, int flags, int device, igb_plan** out);
int igb_plan_counts(const igb_plan* p, long long* n_near, long long* n_far, int* n_nodes);
int igb_plan_near_pairs(const igb_plan* p, int* out);
int igb_plan_far_pairs(const igb_plan* p, int* out);
/* counts[0] = ordered regular near pairs, counts[1..3] = unique singular
 * pairs (vertex, edge, coincident) */
int igb_plan_class_counts(const igb_plan* p, long long counts[4]);
/* cluster boxes (ClusterTree, h2.cpp:49-78; leaves = the element boxes of
 * spaces.cpp:117-147): out[node][6] = min xyz, max xyz.  A plan created on a
 * device computes them there (with the traversal and the pair classes). */
int igb_plan_node_boxes(const igb_plan* p, double* out);
/* row-cluster partition over `world` ranks: rank owns the contiguous range
 * [*c0, *c1) of level-1 clusters (cluster = 4*patch + sx + 2*sy), i.e. the
 * block rows of their leaf elements; reports owned elements and the near /
 * far pairs whose test element / target node lies in them */
int igb_plan_partition(const igb_plan* p, int world, int rank, int* c0, int* c1, int* n_elements,
                       long long* n_near, long long* n_far);
/* ownership masks of that rank: element_owned[ne], node_owned[n_nodes]
 * (roots are owned by every rank) */
int igb_plan_owned(const igb_plan* p, int world, int rank, unsigned char* element_owned, unsigned char* node_owned);
/* Singular items (class >= 1, ea <= eb) of rank `rank` enumerated from the mesh
   topology alone (what the device integrates before the partition exists):
   counts[c] per class, *mismatch = 1 unless they equal the near list's singular
   pairs of build_local_plan (spaces.cpp:309-394 classes over h2.cpp:175-252). */
int igb_plan_singular_items(const igb_plan* p, int world, int rank, long long counts[4], int* mismatch);
void igb_plan_destroy(igb_plan* p);

/* ---- around the operator ---- */
/* SolverOptions / SolveStats (solver.hpp:37-48) */
typedef struct {
  double tol;
  int max_iter;
  int restart;
} igb_solver_opts;
typedef struct {
  int iterations;
  double residual;
  int converged;
  double seconds;
} igb_solve_stats;
/* gmres(LinearOperator{h.apply}, b) (solver.hpp:54-155) and cg (159-200),
 * device-resident vectors; b, x host buffers of rows() scalars */
int igb_h2_gmres(igb_h2* h, const double* b, double* x, const igb_solver_opts* opts, igb_solve_stats* stats);
int igb_h2_cg(igb_h2* h, const double* b, double* x, const igb_solver_opts* opts, igb_solve_stats* stats);
/* load vectors (assembly.cpp:55-133): the quadrature points of every element
 * (element-major, *n_per_element points each, xyz), then b from the data
 * values at those points (one Scalar per point; Maxwell: 3 complex) */
int igb_rhs_points(const igb_discretization* d, int quad_order, int device, double* pts, int* n_per_element);
int igb_rhs_assemble(const igb_discretization* d, int quad_order, int device, const double* values, double* b);
/* eval_potential / eval_maxwell_potential (operators.cpp:112-208); out: one
 * Scalar per point, Maxwell 3 complex per point */
int igb_potential(const igb_discretization* d, const double* density, int n_points, const double* points,
                  int quad_order, int device, double* out);
/* assemble_dense / assemble_dense_complex (assembly.cpp:16-53, assembly.hpp:25-28):
 * the dense Galerkin matrix on the device, `out` = host, column-major
 * dof_count x dof_count Scalar (Eigen MatrixXd / MatrixXcd memory); orders 0 ->
 * P+2 / P+3 as AssemblyOptions */
int igb_dense_assemble(const igb_discretization* d, int far_order, int sing_order, int device, double* out);

/* eta-admissibility of two boxes (min xyz, max xyz), h2.cpp:92-97 */
int igb_admissible(const double box_a[6], const double box_b[6], double eta);
int igb_last_error(char* buf, size_t n);
int igb_version(void);
/* device memory of destroyed operators stays reserved in a per-device pool for
 * the next construction (bounded by IGB_POOL_KEEP_MB); this returns it to the
 * driver (e.g. before handing the device to another allocator).  No reference
 * counterpart: the reference holds its operator in host memory. */
int igb_release_device_memory(int device);

#ifdef __cplusplus
}
#endif

#endif /* IGABEM_B200_H */
