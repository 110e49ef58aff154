// C ABI (include/igabem_b200.h) over the host model and the device operator.
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>

#include "../../include/igabem_b200.h"
#include "igb_apps.hpp"
#include "igb_device.hpp"
#include "igb_host.hpp"

struct igb_geometry {
  std::shared_ptr<const igb::Geometry> g;
};
struct igb_discretization {
  std::shared_ptr<const igb::Discretization> d;
};
struct igb_h2 {
  std::unique_ptr<igb::H2Device> dev;
};
struct igb_plan {
  std::shared_ptr<const igb::Discretization> d;
  igb::H2Plan plan;
};

namespace {
thread_local std::string g_err;

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return IGB_OK;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return IGB_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return IGB_DOMAIN_ERROR;
  } catch (const std::logic_error& e) {
    g_err = e.what();
    return IGB_LOGIC_ERROR;
  } catch (const std::runtime_error& e) {
    g_err = e.what();
    return std::strncmp(e.what(), "CUDA error", 10) == 0 ? IGB_CUDA_ERROR : IGB_RUNTIME_ERROR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return IGB_RUNTIME_ERROR;
  }
}
void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string("null argument: ") + what);
}
}  // namespace

extern "C" {

int igb_version(void) { return 1; }

int igb_last_error(char* buf, size_t n) {
  if (buf && n) std::snprintf(buf, n, "%s", g_err.c_str());
  return static_cast<int>(g_err.size());
}

int igb_geometry_create(int n_patches, const igb_patch_desc* patches, igb_geometry** out) {
  return guard([&] {
    need(out, "out");
    if (n_patches < 1) throw std::invalid_argument("Geometry: no patches");
    need(patches, "patches");
    std::vector<igb::Patch> ps;
    for (int i = 0; i < n_patches; ++i) {
      const igb_patch_desc& d = patches[i];
      need(d.knots_u, "knots_u");
      need(d.knots_v, "knots_v");
      need(d.ctrl_w, "ctrl_w");
      need(d.weight, "weight");
      igb::Patch p;
      p.kv_u = igb::make_knots(std::vector<double>(d.knots_u, d.knots_u + d.n_knots_u), d.degree_u);
      p.kv_v = igb::make_knots(std::vector<double>(d.knots_v, d.knots_v + d.n_knots_v), d.degree_v);
      const int n = p.count_u() * p.count_v();
      p.cw.assign(d.ctrl_w, d.ctrl_w + 3 * n);
      p.w.assign(d.weight, d.weight + n);
      ps.push_back(std::move(p));
    }
    *out = new igb_geometry{std::make_shared<igb::Geometry>(std::move(ps))};
  });
}
int igb_geometry_sphere(double radius, const double center[3], igb_geometry** out) {
  return guard([&] {
    need(out, "out");
    const igb::V3 c = center ? igb::V3(center[0], center[1], center[2]) : igb::V3();
    *out = new igb_geometry{igb::make_sphere(radius, c)};
  });
}
int igb_geometry_square(igb_geometry** out) {
  return guard([&] {
    need(out, "out");
    *out = new igb_geometry{igb::make_square()};
  });
}
int igb_geometry_info(const igb_geometry* g, int* n_patches, int* n_edges, int* n_vertices) {
  return guard([&] {
    need(g, "geometry");
    if (n_patches) *n_patches = g->g->patch_count();
    if (n_edges) *n_edges = static_cast<int>(g->g->edges().size());
    if (n_vertices) *n_vertices = static_cast<int>(g->g->vertices().size());
  });
}
void igb_geometry_destroy(igb_geometry* g) { delete g; }

int igb_discretization_create(const igb_geometry* g, int kind, double kre, double kim, int degree, int rep,
                              int level, igb_discretization** out) {
  return guard([&] {
    need(g, "geometry");
    need(out, "out");
    *out = new igb_discretization{
        std::make_shared<igb::Discretization>(g->g, kind, igb::cplx(kre, kim), degree, rep, level)};
  });
}
int igb_discretization_info(const igb_discretization* d, igb_disc_info* o) {
  return guard([&] {
    need(d, "discretization");
    need(o, "out");
    const auto& x = *d->d;
    o->dof_count = x.dof_count();
    o->element_count = x.element_count();
    o->local_count = x.local_count();
    o->level = x.level();
    o->degree = x.degree();
    o->repetition = x.repetition();
    o->kind = x.kind();
    o->patch_count = x.geometry().patch_count();
  });
}
int igb_discretization_l2g(const igb_discretization* d, int* l2g, double* sign) {
  return guard([&] {
    need(d, "discretization");
    const auto& x = *d->d;
    if (l2g) std::memcpy(l2g, x.l2g().data(), x.l2g().size() * sizeof(int));
    if (sign) std::memcpy(sign, x.lsign().data(), x.lsign().size() * sizeof(double));
  });
}
int igb_discretization_elements(const igb_discretization* d, int* ints, double* dbl) {
  return guard([&] {
    need(d, "discretization");
    const auto& x = *d->d;
    for (int e = 0; e < x.element_count(); ++e) {
      const auto& el = x.element(e);
      if (ints) {
        ints[3 * e] = el.patch;
        ints[3 * e + 1] = el.ix;
        ints[3 * e + 2] = el.iy;
      }
      if (dbl) {
        double* o = dbl + 9 * e;
        o[0] = el.h;
        o[1] = el.ox;
        o[2] = el.oy;
        for (int k = 0; k < 3; ++k) {
          o[3 + k] = el.box.mn[k];
          o[6 + k] = el.box.mx[k];
        }
      }
    }
  });
}
int igb_classify_pair(const igb_discretization* d, int ea, int eb, int* cls, int maps[6]) {
  return guard([&] {
    need(d, "discretization");
    const auto& x = *d->d;
    if (ea < 0 || eb < 0 || ea >= x.element_count() || eb >= x.element_count())
      throw std::invalid_argument("classify_pair: element index out of range");
    const igb::PairInfo info = x.classify_pair(ea, eb);
    if (cls) *cls = info.cls;
    if (maps) {
      maps[0] = info.map_a.swap;
      maps[1] = info.map_a.flip_u;
      maps[2] = info.map_a.flip_v;
      maps[3] = info.map_b.swap;
      maps[4] = info.map_b.flip_u;
      maps[5] = info.map_b.flip_v;
    }
  });
}
void igb_discretization_destroy(igb_discretization* d) { delete d; }

int igb_h2_create(const igb_discretization* d, const igb_h2_opts* opts, int device, igb_h2** out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb_h2_opts o = opts ? *opts : igb_h2_opts{8, 1.6, 0, 0};
    *out = new igb_h2{std::make_unique<igb::H2Device>(d->d, o.m, o.eta, o.far_order, o.sing_order, device)};
  });
}
int igb_h2_create_ex(const igb_discretization* d, const igb_h2_opts* opts, int device, int flags, igb_h2** out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb_h2_opts o = opts ? *opts : igb_h2_opts{8, 1.6, 0, 0};
    *out = new igb_h2{std::make_unique<igb::H2Device>(d->d, o.m, o.eta, o.far_order, o.sing_order, device, flags)};
  });
}
int igb_h2_create_dist(const igb_discretization* d, const igb_h2_opts* opts, int device, int flags, int world,
                       int rank, igb_h2** out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb_h2_opts o = opts ? *opts : igb_h2_opts{8, 1.6, 0, 0};
    *out = new igb_h2{
        std::make_unique<igb::H2Device>(d->d, o.m, o.eta, o.far_order, o.sing_order, device, flags, world, rank)};
  });
}
int igb_h2_dist_send_count(const igb_h2* h, size_t* scalars) {
  return guard([&] {
    need(h, "h2");
    need(scalars, "scalars");
    *scalars = h->dev->send_count();
  });
}
int igb_h2_dist_dof_mask(const igb_h2* h, unsigned char* mask) {
  return guard([&] {
    need(h, "h2");
    need(mask, "mask");
    const auto& ds = h->dev->local_plan().dof_start;
    for (size_t i = 0; i + 1 < ds.size(); ++i) mask[i] = ds[i + 1] > ds[i] ? 1 : 0;
  });
}
int igb_h2_dist_phase1(igb_h2* h, const double* x, double* send, void* stream) {
  return guard([&] {
    need(h, "h2");
    need(x, "x");
    h->dev->dist_phase1(x, send, static_cast<cudaStream_t>(stream));
  });
}
int igb_h2_dist_phase2(igb_h2* h, const double* recv, double* y, void* stream) {
  return guard([&] {
    need(h, "h2");
    need(y, "y");
    h->dev->dist_phase2(recv, y, static_cast<cudaStream_t>(stream));
  });
}
int igb_h2_dim(const igb_h2* h, int* rows) {
  return guard([&] {
    need(h, "h2");
    need(rows, "rows");
    *rows = h->dev->dim();
  });
}
int igb_h2_apply(igb_h2* h, const double* x, double* y) {
  return guard([&] {
    need(h, "h2");
    need(x, "x");
    need(y, "y");
    h->dev->apply_host(x, y);
  });
}
int igb_h2_apply_device(igb_h2* h, const double* x, double* y, void* stream) {
  return guard([&] {
    need(h, "h2");
    need(x, "x");
    need(y, "y");
    h->dev->apply_device(x, y, static_cast<cudaStream_t>(stream));
  });
}
int igb_h2_storage_report(const igb_h2* h, igb_h2_storage* o) {
  return guard([&] {
    need(h, "h2");
    need(o, "out");
    const auto& P = h->dev->plan();
    const size_t nl = h->dev->disc().local_count(), mm = static_cast<size_t>(P.m) * P.m;
    const size_t s = h->dev->is_complex() ? 16 : 8;
    o->nearfield_entries = P.near_a.size() * nl * nl;
    o->farfield_entries = P.far_a.size() * mm * mm;
    const size_t mom = static_cast<size_t>(h->dev->disc().element_count()) * h->dev->nch() * mm * nl;
    o->total_bytes = (o->nearfield_entries + o->farfield_entries + mom + 2 * static_cast<size_t>(P.m) * P.m) * s;
  });
}
int igb_h2_counts(const igb_h2* h, long long* n_near, long long* n_far, int* n_nodes) {
  return guard([&] {
    need(h, "h2");
    const auto& P = h->dev->plan();
    if (n_near) *n_near = static_cast<long long>(P.near_a.size());
    if (n_far) *n_far = static_cast<long long>(P.far_a.size());
    if (n_nodes) *n_nodes = P.n_nodes;
  });
}
int igb_h2_near_pairs(const igb_h2* h, int* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    const auto& P = h->dev->plan();
    for (size_t i = 0; i < P.near_a.size(); ++i) {
      out[2 * i] = P.near_a[i];
      out[2 * i + 1] = P.near_b[i];
    }
  });
}
int igb_h2_far_pairs(const igb_h2* h, int* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    const auto& P = h->dev->plan();
    for (size_t i = 0; i < P.far_a.size(); ++i) {
      out[2 * i] = P.far_a[i];
      out[2 * i + 1] = P.far_b[i];
    }
  });
}
int igb_h2_tree(const igb_h2* h, int* patch, int* level, int* sx, int* sy, double* boxes) {
  return guard([&] {
    need(h, "h2");
    const auto& P = h->dev->plan();
    for (int i = 0; i < P.n_nodes; ++i) {
      if (patch) patch[i] = P.node_patch[i];
      if (level) level[i] = P.node_level[i];
      if (sx) sx[i] = P.node_sx[i];
      if (sy) sy[i] = P.node_sy[i];
      if (boxes)
        for (int k = 0; k < 3; ++k) {
          boxes[6 * i + k] = P.node_box[i].mn[k];
          boxes[6 * i + 3 + k] = P.node_box[i].mx[k];
        }
    }
  });
}
int igb_h2_near_blocks(const igb_h2* h, long long first, long long count, double* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    h->dev->near_blocks(first, count, out);
  });
}
int igb_h2_couplings(const igb_h2* h, long long first, long long count, double* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    h->dev->couplings(first, count, out);
  });
}
int igb_h2_moments(const igb_h2* h, double* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    h->dev->moments(out);
  });
}
int igb_h2_images(const igb_h2* h, double* out) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    h->dev->images(out);
  });
}
int igb_h2_assembly_times(const igb_h2* h, igb_h2_times* o) {
  return guard([&] {
    need(h, "h2");
    need(o, "out");
    const auto& t = h->dev->times();
    o->plan_host_ms = t.plan_host;
    o->upload_ms = t.upload;
    o->elements_ms = t.elements;
    o->images_ms = t.images;
    o->couplings_ms = t.couplings;
    o->regular_ms = t.regular;
    o->coincident_ms = t.singular[3];
    o->edge_ms = t.singular[2];
    o->vertex_ms = t.singular[1];
    o->device_total_ms = t.total_device;
    o->wall_total_ms = t.total_wall;
    o->scatter_ms = t.scatter;
  });
}
int igb_h2_device_bytes(const igb_h2* h, size_t* near, size_t* far, size_t* moments) {
  return guard([&] {
    need(h, "h2");
    const auto b = h->dev->bytes();
    if (near) *near = b.near;
    if (far) *far = b.far;
    if (moments) *moments = b.moments;
  });
}
int igb_h2_bench_apply(igb_h2* h, int iters, float* ms, int* launches) {
  return guard([&] {
    need(h, "h2");
    cudaSetDevice(h->dev->device());
    cudaStream_t s = h->dev->stream();
    h->dev->launch_apply_graph(s);  // instantiate outside the timed region
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, s);
    for (int i = 0; i < iters; ++i) h->dev->launch_apply_graph(s);
    cudaEventRecord(b, s);
    const cudaError_t err = cudaEventSynchronize(b);
    float t = 0;
    cudaEventElapsedTime(&t, a, b);
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    if (err != cudaSuccess) throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(err));
    if (ms) *ms = t;
    if (launches) *launches = h->dev->apply_kernel_launches();
  });
}
int igb_h2_reassemble(igb_h2* h, double* device_ms, int* launches) {
  return guard([&] {
    need(h, "h2");
    const double ms = h->dev->reassemble();
    if (device_ms) *device_ms = ms;
    if (launches) *launches = h->dev->assembly_kernel_launches();
  });
}
int igb_h2_profile_kernels(igb_h2* h, int iters, int max_n, char* names, double* ms, int* n) {
  return guard([&] {
    need(h, "h2");
    need(n, "n");
    const auto k = h->dev->profile_kernels(iters);
    *n = static_cast<int>(std::min<size_t>(k.size(), static_cast<size_t>(std::max(max_n, 0))));
    for (int i = 0; i < *n; ++i) {
      if (names) std::snprintf(names + 32 * i, 32, "%s", k[i].first.c_str());
      if (ms) ms[i] = k[i].second;
    }
  });
}
int igb_h2_far_field(igb_h2* h, const double* x, double* up, double* down) {
  return guard([&] {
    need(h, "h2");
    need(x, "x");
    h->dev->far_field(x, up, down);
  });
}
int igb_h2_far_work(const igb_h2* h, long long pairs[2]) {
  return guard([&] {
    need(h, "h2");
    need(pairs, "pairs");
    pairs[0] = h->dev->sym_pairs(0);
    pairs[1] = h->dev->sym_pairs(1);
  });
}
int igb_h2_leaf_blocks(const igb_h2* h, long long out[3]) {
  return guard([&] {
    need(h, "h2");
    need(out, "out");
    out[0] = h->dev->leaf_block_pairs();
    out[1] = static_cast<long long>(h->dev->leaf_block_bytes());
    out[2] = static_cast<long long>(h->dev->block_stream_bytes());
  });
}
int igb_h2_profile_apply(igb_h2* h, int iters, double phase_ms[8]) {
  return guard([&] {
    need(h, "h2");
    need(phase_ms, "phase_ms");
    h->dev->profile_apply(iters, phase_ms);
  });
}
int igb_h2_bench_steps(igb_h2* h, int steps, int matvecs, double* total_ms, double* assembly_ms) {
  return guard([&] {
    need(h, "h2");
    const double t = h->dev->bench_steps(steps, matvecs, assembly_ms);
    if (total_ms) *total_ms = t;
  });
}
int igb_h2_class_counts(const igb_h2* h, long long counts[4]) {
  return guard([&] {
    need(h, "h2");
    need(counts, "counts");
    const auto& P = h->dev->plan();
    counts[0] = static_cast<long long>(P.reg_slot.size());
    for (int c = 1; c <= 3; ++c) counts[c] = static_cast<long long>(P.sing[c].ea.size());
  });
}
int igb_h2_launch_counts(const igb_h2* h, int* assembly, int* apply) {
  return guard([&] {
    need(h, "h2");
    if (assembly) *assembly = h->dev->assembly_kernel_launches();
    if (apply) *apply = h->dev->apply_kernel_launches();
  });
}
int igb_h2_upload_bytes(const igb_h2* h, size_t* bytes) {
  return guard([&] {
    need(h, "h2");
    need(bytes, "bytes");
    *bytes = h->dev->upload_bytes();
  });
}
void igb_h2_destroy(igb_h2* h) { delete h; }

int igb_plan_create(const igb_discretization* d, const igb_h2_opts* opts, igb_plan** out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb_h2_opts o = opts ? *opts : igb_h2_opts{8, 1.6, 0, 0};
    auto p = std::make_unique<igb_plan>();
    p->d = d->d;
    p->plan = igb::build_plan(*d->d, o.m, o.eta, o.far_order, o.sing_order);
    *out = p.release();
  });
}
int igb_plan_create_ex(const igb_discretization* d, const igb_h2_opts* opts, int flags, int device, igb_plan** out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb_h2_opts o = opts ? *opts : igb_h2_opts{8, 1.6, 0, 0};
    auto p = std::make_unique<igb_plan>();
    p->d = d->d;
    p->plan = igb::build_plan(*d->d, o.m, o.eta, o.far_order, o.sing_order, (flags & 4) ? device : -1);
    *out = p.release();
  });
}
int igb_plan_counts(const igb_plan* p, long long* n_near, long long* n_far, int* n_nodes) {
  return guard([&] {
    need(p, "plan");
    if (n_near) *n_near = static_cast<long long>(p->plan.near_a.size());
    if (n_far) *n_far = static_cast<long long>(p->plan.far_a.size());
    if (n_nodes) *n_nodes = p->plan.n_nodes;
  });
}
int igb_plan_near_pairs(const igb_plan* p, int* out) {
  return guard([&] {
    need(p, "plan");
    need(out, "out");
    for (size_t i = 0; i < p->plan.near_a.size(); ++i) {
      out[2 * i] = p->plan.near_a[i];
      out[2 * i + 1] = p->plan.near_b[i];
    }
  });
}
int igb_plan_far_pairs(const igb_plan* p, int* out) {
  return guard([&] {
    need(p, "plan");
    need(out, "out");
    for (size_t i = 0; i < p->plan.far_a.size(); ++i) {
      out[2 * i] = p->plan.far_a[i];
      out[2 * i + 1] = p->plan.far_b[i];
    }
  });
}
int igb_plan_class_counts(const igb_plan* p, long long counts[4]) {
  return guard([&] {
    need(p, "plan");
    need(counts, "counts");
    counts[0] = static_cast<long long>(p->plan.reg_slot.size());
    for (int c = 1; c <= 3; ++c) counts[c] = static_cast<long long>(p->plan.sing[c].ea.size());
  });
}
int igb_plan_node_boxes(const igb_plan* p, double* out) {
  return guard([&] {
    need(p, "plan");
    need(out, "out");
    for (size_t i = 0; i < p->plan.node_box.size(); ++i)
      for (int k = 0; k < 3; ++k) {
        out[6 * i + k] = p->plan.node_box[i].mn[k];
        out[6 * i + 3 + k] = p->plan.node_box[i].mx[k];
      }
  });
}
int igb_plan_partition(const igb_plan* p, int world, int rank, int* c0, int* c1, int* n_elements,
                       long long* n_near, long long* n_far) {
  return guard([&] {
    need(p, "plan");
    const auto r = igb::partition_rows(*p->d, p->plan, world, rank);
    if (c0) *c0 = r.c0;
    if (c1) *c1 = r.c1;
    if (n_elements) *n_elements = static_cast<int>(r.elements.size());
    if (n_near) *n_near = r.near_count;
    if (n_far) *n_far = r.far_count;
  });
}
int igb_plan_owned(const igb_plan* p, int world, int rank, unsigned char* element_owned, unsigned char* node_owned) {
  return guard([&] {
    need(p, "plan");
    const auto lp = igb::build_local_plan(*p->d, p->plan, world, rank);
    if (element_owned)
      for (size_t e = 0; e < lp.el_local.size(); ++e) element_owned[e] = lp.el_local[e] >= 0 ? 1 : 0;
    if (node_owned) std::copy(lp.node_owned.begin(), lp.node_owned.end(), node_owned);
  });
}
int igb_plan_singular_items(const igb_plan* p, int world, int rank, long long counts[4], int* mismatch) {
  return guard([&] {
    need(p, "plan");
    std::vector<unsigned char> own;
    if (world > 1) own = igb::owned_elements(*p->d, world, rank);
    igb::SingList items[4];
    p->d->singular_items(own.empty() ? nullptr : own.data(), items);
    const auto lp = igb::build_local_plan(*p->d, p->plan, world, rank);
    int bad = 0;
    for (int c = 1; c <= 3; ++c) {
      const auto &T = items[c], &L = lp.sing[c];
      bad |= T.ea != L.ea || T.eb != L.eb || T.map_a != L.map_a || T.map_b != L.map_b;
    }
    if (counts) {
      counts[0] = static_cast<long long>(lp.reg_slot.size());
      for (int c = 1; c <= 3; ++c) counts[c] = static_cast<long long>(items[c].ea.size());
    }
    if (mismatch) *mismatch = bad;
  });
}
void igb_plan_destroy(igb_plan* p) { delete p; }

int igb_h2_gmres(igb_h2* h, const double* b, double* x, const igb_solver_opts* opts, igb_solve_stats* stats) {
  return guard([&] {
    need(h, "h2");
    need(b, "b");
    need(x, "x");
    igb::SolverOpts o;
    if (opts) o = igb::SolverOpts{opts->tol, opts->max_iter, opts->restart};
    const auto r = igb::gmres(*h->dev, b, x, o);
    if (stats) *stats = igb_solve_stats{r.iterations, r.residual, r.converged ? 1 : 0, r.seconds};
  });
}
int igb_h2_cg(igb_h2* h, const double* b, double* x, const igb_solver_opts* opts, igb_solve_stats* stats) {
  return guard([&] {
    need(h, "h2");
    need(b, "b");
    need(x, "x");
    igb::SolverOpts o;
    if (opts) o = igb::SolverOpts{opts->tol, opts->max_iter, opts->restart};
    const auto r = igb::cg(*h->dev, b, x, o);
    if (stats) *stats = igb_solve_stats{r.iterations, r.residual, r.converged ? 1 : 0, r.seconds};
  });
}
int igb_rhs_points(const igb_discretization* d, int quad_order, int device, double* pts, int* n_per_element) {
  return guard([&] {
    need(d, "discretization");
    const int n = quad_order > 0 ? quad_order : d->d->degree() + 2;
    if (n_per_element) *n_per_element = n * n;
    if (pts) {
      std::vector<double> v;
      igb::quad_points(*d->d, quad_order, device, v);
      std::memcpy(pts, v.data(), v.size() * sizeof(double));
    }
  });
}
int igb_rhs_assemble(const igb_discretization* d, int quad_order, int device, const double* values, double* b) {
  return guard([&] {
    need(d, "discretization");
    need(values, "values");
    need(b, "b");
    igb::assemble_rhs(*d->d, quad_order, device, values, b);
  });
}
int igb_potential(const igb_discretization* d, const double* density, int n_points, const double* points,
                  int quad_order, int device, double* out) {
  return guard([&] {
    need(d, "discretization");
    need(density, "density");
    if (n_points < 0) throw std::invalid_argument("eval_potential: negative point count");
    igb::eval_potential(*d->d, quad_order, device, density, n_points, points, out);
  });
}

int igb_dense_assemble(const igb_discretization* d, int far_order, int sing_order, int device, double* out) {
  return guard([&] {
    need(d, "discretization");
    need(out, "out");
    igb::dense_assemble(*d->d, far_order, sing_order, device, out);
  });
}

int igb_release_device_memory(int device) {
  return guard([&] { igb::release_device_memory(device); });
}

int igb_admissible(const double a[6], const double b[6], double eta) {
  igb::Box A, B;
  for (int k = 0; k < 3; ++k) {
    A.mn[k] = a[k];
    A.mx[k] = a[3 + k];
    B.mn[k] = b[k];
    B.mx[k] = b[3 + k];
  }
  const double da = A.diag_norm(), db = B.diag_norm();
  return std::max(da, db) <= eta * A.exterior_distance(B) ? 1 : 0;
}

}  // extern "C"
