// Host-side model of the reference's Geometry / Discretization / ClusterTree
// (igabem: proj/core/include/igabem/{splines,geometry,spaces,h2}.hpp), laid
// out as flat arrays for upload to the B200.  This is setup code around the
// hot path: element boxes, the cluster tree, the admissibility traversal and
// pair classification run here (OpenMP); every floating-point operation that
// decides the block partition rounds exactly like the reference so the
// partition is bit-identical.
#pragma once

#include <array>
#include <complex>
#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace igb {

using cplx = std::complex<double>;

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
inline V3 operator/(const V3& a, double s) { return {a[0] / s, a[1] / s, a[2] / s}; }
inline double dot(const V3& a, const V3& b) { return a[0] * b[0] + a[1] * b[1] + a[2] * b[2]; }
inline double norm(const V3& a) { return __builtin_sqrt(dot(a, a)); }
inline V3 cross(const V3& a, const V3& b) {
  return {a[1] * b[2] - a[2] * b[1], a[2] * b[0] - a[0] * b[2], a[0] * b[1] - a[1] * b[0]};
}

// Axis-aligned box with Eigen::AlignedBox3d semantics.
struct Box {
  double mn[3], mx[3];
  void set_empty();
  void extend(const V3& p);
  void extend(const Box& b);
  double diag_norm() const;
  double exterior_distance(const Box& b) const;
};

// Clamped knot vector (splines.hpp:11-31).
struct KnotVector {
  std::vector<double> knots;
  int degree = 0;
  int size() const { return static_cast<int>(knots.size()) - degree - 1; }
  int find_span(double x) const;
};
KnotVector make_knots(std::vector<double> k, int p);
KnotVector make_uniform_knots(int p, int level, int rep);

// NURBS patch with homogeneous control points (splines.hpp:53-67).
struct Patch {
  KnotVector kv_u, kv_v;
  std::vector<double> cw;  // 3 per control point, index i + j*count_u
  std::vector<double> w;
  int count_u() const { return kv_u.size(); }
  int count_v() const { return kv_v.size(); }
  V3 point(int i, int j) const;
};
struct Jet {
  V3 x, du, dv;
};
Jet eval_patch(const Patch& s, double u, double v);  // splines.cpp:183-216

struct EdgeIdent {
  int patch_a, edge_a, patch_b, edge_b;
  bool reversed;
};
struct VertexIdent {
  int patch_a, corner_a, patch_b, corner_b;
};

// Multi-patch geometry (geometry.hpp:38-76).
class Geometry {
 public:
  explicit Geometry(std::vector<Patch> patches);
  int patch_count() const { return static_cast<int>(patches_.size()); }
  const Patch& patch(int i) const { return patches_[i]; }
  const std::vector<EdgeIdent>& edges() const { return edges_; }
  const std::vector<VertexIdent>& vertices() const { return vertices_; }
  double check_matching() const;  // max deviation over violating edge pairs, 0 if none
 private:
  std::vector<Patch> patches_;
  std::vector<EdgeIdent> edges_;
  std::vector<VertexIdent> vertices_;
};
std::shared_ptr<Geometry> make_sphere(double radius, const V3& center);  // shapes.cpp:87-205
std::shared_ptr<Geometry> make_square();                                  // shapes.cpp:28-30

enum Kind { kLaplace = 0, kHelmholtz = 1, kMaxwell = 2 };
enum PairClass { kFar = 0, kVertex = 1, kEdge = 2, kCoincident = 3 };

struct SquareMap {
  bool swap = false, flip_u = false, flip_v = false;
  int bits() const { return (swap ? 1 : 0) | (flip_u ? 2 : 0) | (flip_v ? 4 : 0); }
};
struct PairInfo {
  int cls = kFar;
  SquareMap map_a, map_b;
};

struct Element {
  int patch, ix, iy;
  double h, ox, oy;
  Box box;
};

// Power-basis form of one patch knot-span cell: homogeneous (wx, wy, wz, w)
// as polynomials in (u - u0, v - v0); coef[c][j][i] multiplies s^i t^j.
constexpr int kMaxGeomDeg = 4;
struct GeomCell {
  double u0, v0;
  double coef[4][kMaxGeomDeg + 1][kMaxGeomDeg + 1];
};

// Unique singular work items of one class (ea <= eb): element ids, map bits
// and, once a block partition exists, the two near-list output slots (slot of
// (ea,eb) and of (eb,ea); equal for coincident pairs).
struct SingList {
  std::vector<int> ea, eb, slot_ab, slot_ba;
  std::vector<uint8_t> map_a, map_b;
};

// Discrete space (spaces.hpp:37-105).
class Discretization {
 public:
  Discretization(std::shared_ptr<const Geometry> g, int kind, cplx kappa, int degree, int rep,
                 int level);
  const Geometry& geometry() const { return *geom_; }
  int kind() const { return kind_; }
  cplx kappa() const { return kappa_; }
  bool is_complex() const { return kind_ != kLaplace; }
  bool is_vector() const { return kind_ == kMaxwell; }
  int degree() const { return degree_; }
  int repetition() const { return rep_; }
  int level() const { return level_; }
  int dof_count() const { return n_dofs_; }
  int element_count() const { return static_cast<int>(elements_.size()); }
  int local_count() const { return n_local_; }
  int elements_per_patch() const { return epp_; }
  const Element& element(int e) const { return elements_[e]; }
  int element_index(int p, int ix, int iy) const { return p * epp_ + ix + (1 << level_) * iy; }
  const std::vector<int>& l2g() const { return l2g_; }
  const std::vector<double>& lsign() const { return lsign_; }
  PairInfo classify_pair(int ea, int eb) const;
  // patch-pair topology tables of classify_pair, flattened for the device
  // classification (igb_plan_gpu.cu): CSR over (patch a, patch b) of shared
  // edges {edge_a, edge_b, reversed} and shared corners {corner_a, corner_b},
  // in classify_pair's iteration order
  void flatten_topology(std::vector<int>& edge_rs, std::vector<int>& edges, std::vector<int>& corner_rs,
                        std::vector<int>& corners) const;
 // spaces.cpp:309-394
  // The singular items (classify_pair class >= 1, ea <= eb) enumerated from the
  // mesh topology alone -- no block tree: same-patch neighbours, elements along
  // shared patch edges and at shared patch corners.  Ascending (ea, eb): the
  // order build_plan extracts them from the sorted near list.  owned != null:
  // only items with ea or eb owned (a rank's block rows).  No slots.
  void singular_items(const unsigned char* owned, SingList out[4]) const;

  // GPU tables ---------------------------------------------------------
  // geometry cells and per-element cell index
  const std::vector<GeomCell>& cells() const { return cells_; }
  const std::vector<int>& element_cell() const { return element_cell_; }
  int geom_degree() const { return geom_degree_; }
  // 1D local basis polynomials per grid position: [pos][fn][power], in the
  // element-local coordinate s in [0,1] (u = origin + h s).
  // scalar space: degree q = scalar_degree(); Maxwell: degree P (tab_p) and
  // P-1 (tab_q).
  int scalar_degree() const { return scalar_q_; }
  const std::vector<double>& tab_s() const { return tab_s_; }
  const std::vector<double>& tab_p() const { return tab_p_; }
  const std::vector<double>& tab_q() const { return tab_q_; }

 private:
  void build_elements();
  void build_scalar();
  void build_maxwell();
  void build_cells();
  void build_tables();

  std::shared_ptr<const Geometry> geom_;
  int kind_;
  cplx kappa_;
  int degree_, rep_, level_;
  int epp_ = 0, n_dofs_ = 0, n_local_ = 0;
  KnotVector scalar_kv_, vec_kv_p_, vec_kv_q_;
  int scalar_q_ = 0;
  std::vector<Element> elements_;
  std::vector<int> l2g_;
  std::vector<double> lsign_;
  struct CrossEdge {
    int edge_a, edge_b;
    bool reversed;
  };
  struct CrossCorner {
    int corner_a, corner_b;
  };
  std::vector<std::vector<std::vector<CrossEdge>>> cross_edges_;
  std::vector<std::vector<std::vector<CrossCorner>>> cross_corners_;
  std::vector<GeomCell> cells_;
  std::vector<int> element_cell_;
  int geom_degree_ = 0;
  std::vector<double> tab_s_, tab_p_, tab_q_;
};

// Rule-independent 1D data.
void gauss_rule(int n, std::vector<double>& nodes, std::vector<double>& weights);  // quadrature.cpp:15-50
std::vector<double> cheb_nodes(int m);                                              // h2.cpp:13-17
void lagrange_all(const std::vector<double>& nodes, double x, double* out);         // h2.cpp:30-45

// Block partition + everything the device assembly / matvec needs that is
// integer bookkeeping (h2.cpp:49-97,175-252).
struct H2Plan {
  int m = 8;
  double eta = 1.6;
  int nfar = 0, nsing = 0;
  int depth = 0, npp = 0, n_nodes = 0, n_patches = 0;
  std::vector<int> level_offset;
  std::vector<int> node_patch, node_level, node_sx, node_sy;
  std::vector<Box> node_box;
  // sorted pair lists
  std::vector<int> near_a, near_b;  // element pairs, sorted by (a, b)
  std::vector<int> far_a, far_b;    // node pairs, sorted by (a, b)
  std::vector<int> near_row_start;  // ne + 1
  std::vector<int> far_row_start;   // n_nodes + 1
  std::vector<int> far_upper_start; // per node: first pair (t, s) of row t with s > t
  std::vector<int> far_trans;       // per pair (t, s): index of (s, t)
  // near pair classification
  std::vector<uint8_t> near_cls;
  // device setup (partition_device >= 0): map bits of the near pairs as classified on the device
  std::vector<uint8_t> dev_map_a, dev_map_b;
  // unique singular work items per class (ea <= eb): element ids, map bits,
  // and the two output slots (slot of (ea,eb) and of (eb,ea); equal for
  // coincident pairs)
  using SingList = igb::SingList;
  SingList sing[4];
  std::vector<int> reg_slot;  // regular near pairs (slot into near list)
  std::vector<int> reg_ab, reg_ba;  // unique regular pairs ea < eb: slots of (ea,eb) and (eb,ea)
  // DOF gather incidence for the deterministic scatter: for dof d the
  // (e*nl + l) entries in ascending order, sign folded in by the device
  std::vector<int> dof_start, dof_inc;
  // interpolation data
  std::vector<double> cheb, tl, tr;  // m, m*m (column-major), m*m

  long long node_id(int p, int l, int sx, int sy) const {
    return static_cast<long long>(p) * npp + level_offset[l] + sx + (1LL << l) * sy;
  }
};
// partition_device >= 0: the traversal, sort, row starts, upper starts and
// transposes run on that CUDA device (device_partition, bit-identical lists)
H2Plan build_plan(const Discretization& d, int m, double eta, int far_order, int sing_order,
                  int partition_device = -1);
// fills near_a/b, near_row_start, far_a/b, far_row_start, far_upper_start,
// far_trans of P (tree and node boxes already built); igb_plan_gpu.cu
// ... and, on the device as well, the element boxes (spaces.cpp:117-147), the tree boxes
// (h2.cpp:49-78), their diagonals and the classification of the near pairs
// (spaces.cpp:309-394): node_box, near_cls, dev_map_a/b
void device_partition(H2Plan& P, const Discretization& d, double eta, int device);
// Option checks of build_plan (h2.hpp:60 ctor) and the quadrature orders it
// derives (far: degree + 2, singular: degree + 3 unless given).
void check_h2_options(const Discretization& d, int m, double eta, int far_order, int sing_order, int* nfar,
                      int* nsing);

// Row-cluster partition: rank owns level-1 clusters [c0, c1)
// (cluster = 4 * patch + sx + 2 * sy); with level 0 the whole operator sits
// on rank 0.  Far pairs are owned by the rank owning the target's level-1
// ancestor; level-0 targets are owned by every rank (replicated, tiny).
struct RowPartition {
  int c0 = 0, c1 = 0;
  std::vector<int> elements;          // owned leaf elements, ascending
  std::vector<unsigned char> owns_element;
  long long near_count = 0, far_count = 0;
};
int node_cluster(const H2Plan& P, int node);  // level-1 cluster of a node, -1 for roots
// element ownership of the row partition (no block tree needed)
std::vector<unsigned char> owned_elements(const Discretization& d, int world, int rank);
RowPartition partition_rows(const Discretization& d, const H2Plan& P, int world, int rank);

// Rank-local view of the plan (identity for world == 1): owned block rows,
// their near slots, singular / regular work items touching them, owned tree
// nodes and far targets, and the pack lists of the up-moment all-gather.
struct LocalPlan {
  int world = 1, rank = 0, c0 = 0, c1 = 0;
  std::vector<int> el;                 // owned elements (global ids, ascending)
  std::vector<int> el_local;           // global -> local element index, -1 if not owned
  std::vector<int> near_rs;            // local rows: slot starts (n_owned + 1)
  std::vector<int> near_row;           // per local slot: local row
  std::vector<int> near_ea, near_eb;   // per local slot: global elements
  std::vector<int> slot_local;         // global slot -> local slot or -1
  H2Plan::SingList sing[4];            // items touching owned rows; slots local or -1
  std::vector<int> reg_slot;           // local slots of owned regular pairs
  std::vector<int> reg_ab, reg_ba;     // unique regular pairs touching owned rows: local slots or -1
  std::vector<unsigned char> node_owned;  // per node (roots owned by every rank)
  std::vector<int> far_targets;        // owned nodes with far pairs (ascending)
  std::vector<int> pack_nodes;         // owned nodes at levels >= 1 (ascending): all-gather payload
  std::vector<std::vector<int>> rank_pack_nodes;  // per rank (for unpacking)
  int pack_max = 0;                    // max payload nodes over ranks
  std::vector<int> dof_start, dof_inc; // gather of owned (local e * nl + l) per DOF
};
LocalPlan build_local_plan(const Discretization& d, const H2Plan& P, int world, int rank);

}  // namespace igb
