// Block partition on the device (setup on the GPU).
//
// The dual traversal of h2.cpp:198-216 runs level by level: every frontier
// pair (same-level nodes a, b) is decided far (admissible, h2.cpp:92-97), near
// (inadmissible leaves) or refined into its 16 child pairs; CUB scans compact
// the three outputs.  The admissibility test reproduces the host's (and the
// reference's) operation order exactly -- diagonals from the host, exterior
// distance with explicit round-to-nearest multiplies/adds and a correctly
// rounded square root, no contraction -- so the partition is bit-identical.
// The pair lists are then radix-sorted by (a, b) (the lexicographic order of
// h2.cpp:215-216), and the CSR row starts, upper starts and transposes of the
// symmetric admissible relation come from binary searches.
#include <cuda_runtime.h>

#include <cub/cub.cuh>

#include <chrono>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "igb_host.hpp"

namespace igb {
namespace {

#define IGB_PCUDA(call)                                                                                    \
  do {                                                                                                     \
    const cudaError_t e_ = (call);                                                                         \
    if (e_ != cudaSuccess) throw std::runtime_error(std::string("CUDA error: ") + cudaGetErrorString(e_)); \
  } while (0)

struct DevBox {
  double mn[3], mx[3];
};

// decision of one same-level pair: 0 far, 1 near (leaf level), 2 refine
__global__ void k_decide(long long n, const int* __restrict__ pa, const int* __restrict__ pb,
                         const DevBox* __restrict__ box, const double* __restrict__ diag, double eta, int leaf,
                         unsigned char* __restrict__ dec, int* __restrict__ is_far, int* __restrict__ is_near,
                         int* __restrict__ is_ref) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int a = pa[i], b = pb[i];
  const DevBox A = box[a], B = box[b];
  double d2 = 0.0;  // Box::exterior_distance, term by term like the host
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    if (A.mn[k] > B.mx[k]) {
      const double aux = __dsub_rn(A.mn[k], B.mx[k]);
      d2 = __dadd_rn(d2, __dmul_rn(aux, aux));
    } else if (B.mn[k] > A.mx[k]) {
      const double aux = __dsub_rn(B.mn[k], A.mx[k]);
      d2 = __dadd_rn(d2, __dmul_rn(aux, aux));
    }
  }
  const double dist = __dsqrt_rn(d2);
  const unsigned char c = fmax(diag[a], diag[b]) <= __dmul_rn(eta, dist) ? 0 : (leaf ? 1 : 2);
  dec[i] = c;
  is_far[i] = c == 0;
  is_near[i] = c == 1;
  is_ref[i] = c == 2;
}

struct Level {
  int npp, off, off_next, side;  // nodes per patch, first node of this / next level, 2^level
};

__global__ void k_emit(long long n, const int* __restrict__ pa, const int* __restrict__ pb,
                       const unsigned char* __restrict__ dec, const int* __restrict__ far_pos,
                       const int* __restrict__ near_pos, const int* __restrict__ ref_pos, Level lv, int epp,
                       int n1, unsigned long long* __restrict__ far_keys, long long far_base,
                       unsigned long long* __restrict__ near_keys, int* __restrict__ na, int* __restrict__ nb) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const int a = pa[i], b = pb[i];
  const unsigned char c = dec[i];
  if (c == 0) {
    far_keys[far_base + far_pos[i]] = (static_cast<unsigned long long>(a) << 32) | static_cast<unsigned>(b);
  } else if (c == 1) {  // leaves -> element ids (p * epp + sx + 2^L sy)
    auto el = [&](int node) {
      const int p = node / lv.npp, r = node % lv.npp - lv.off;
      return p * epp + (r % n1) + n1 * (r / n1);
    };
    near_keys[near_pos[i]] = (static_cast<unsigned long long>(el(a)) << 32) | static_cast<unsigned>(el(b));
  } else {
    auto child = [&](int node, int k) {
      const int p = node / lv.npp, r = node % lv.npp - lv.off;
      const int sx = r % lv.side, sy = r / lv.side;
      return p * lv.npp + lv.off_next + (2 * sx + (k & 1)) + 2 * lv.side * (2 * sy + (k >> 1));
    };
    const long long o = 16LL * ref_pos[i];
    for (int ka = 0; ka < 4; ++ka)
      for (int kb = 0; kb < 4; ++kb) {
        na[o + 4 * ka + kb] = child(a, ka);
        nb[o + 4 * ka + kb] = child(b, kb);
      }
  }
}

// split sorted keys into rows (a) / columns (b)
__global__ void k_split(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ A,
                        int* __restrict__ B) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  A[i] = static_cast<int>(keys[i] >> 32);
  B[i] = static_cast<int>(keys[i] & 0xffffffffu);
}

__device__ __forceinline__ long long lower_bound_key(const unsigned long long* keys, long long n,
                                                     unsigned long long k) {
  long long lo = 0, hi = n;
  while (lo < hi) {
    const long long mid = (lo + hi) >> 1;
    if (keys[mid] < k) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}
// row starts (nrows + 1) and, when upper != nullptr, the first pair of row t with column > t
__global__ void k_rows(int nrows, const unsigned long long* __restrict__ keys, long long n, int* __restrict__ rs,
                       int* __restrict__ upper) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nrows) return;
  rs[r] = static_cast<int>(lower_bound_key(keys, n, static_cast<unsigned long long>(r) << 32));
  if (upper && r < nrows)
    upper[r] = static_cast<int>(
        lower_bound_key(keys, n, (static_cast<unsigned long long>(r) << 32) | static_cast<unsigned>(r + 1)));
}
// position of the transposed pair; -1 if the relation is not symmetric
__global__ void k_trans(long long n, const unsigned long long* __restrict__ keys, int* __restrict__ trans) {
  const long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (i >= n) return;
  const unsigned long long k = keys[i], t = (k << 32) | (k >> 32);
  const long long j = lower_bound_key(keys, n, t);
  trans[i] = (j < n && keys[j] == t) ? static_cast<int>(j) : -1;
}

unsigned blocks(long long n) { return static_cast<unsigned>((n + 255) / 256); }

}  // namespace

void device_partition(H2Plan& P, const Discretization& d, const std::vector<double>& diag, double eta, int device) {
  const int L = P.depth, np = P.n_patches, nn = P.n_nodes, ne = d.element_count();
  const int epp = d.elements_per_patch(), n1 = 1 << L;
  IGB_PCUDA(cudaSetDevice(device));
  cudaStream_t st;
  IGB_PCUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  std::vector<void*> mem;
  auto alloc = [&](size_t bytes) {
    void* p = nullptr;
    IGB_PCUDA(cudaMallocAsync(&p, bytes ? bytes : 8, st));
    mem.push_back(p);
    return p;
  };
  auto release = [&] {
    cudaStreamSynchronize(st);
    for (void* p : mem) cudaFreeAsync(p, st);
    cudaStreamSynchronize(st);
    cudaStreamDestroy(st);
  };
  try {
    std::vector<DevBox> hb(nn);
    for (int i = 0; i < nn; ++i)
      for (int k = 0; k < 3; ++k) {
        hb[i].mn[k] = P.node_box[i].mn[k];
        hb[i].mx[k] = P.node_box[i].mx[k];
      }
    DevBox* dbox = static_cast<DevBox*>(alloc(nn * sizeof(DevBox)));
    double* ddiag = static_cast<double*>(alloc(nn * sizeof(double)));
    IGB_PCUDA(cudaMemcpyAsync(dbox, hb.data(), nn * sizeof(DevBox), cudaMemcpyHostToDevice, st));
    IGB_PCUDA(cudaMemcpyAsync(ddiag, diag.data(), nn * sizeof(double), cudaMemcpyHostToDevice, st));
    // level-0 frontier: every ordered root pair
    std::vector<int> ha, hbv;
    for (int a = 0; a < np; ++a)
      for (int b = 0; b < np; ++b) {
        ha.push_back(static_cast<int>(P.node_id(a, 0, 0, 0)));
        hbv.push_back(static_cast<int>(P.node_id(b, 0, 0, 0)));
      }
    long long n = static_cast<long long>(ha.size());
    int* fa = static_cast<int*>(alloc(n * sizeof(int)));
    int* fb = static_cast<int*>(alloc(n * sizeof(int)));
    IGB_PCUDA(cudaMemcpyAsync(fa, ha.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    IGB_PCUDA(cudaMemcpyAsync(fb, hbv.data(), n * sizeof(int), cudaMemcpyHostToDevice, st));
    std::vector<unsigned long long*> far_chunks;
    std::vector<long long> far_counts;
    unsigned long long* near_keys = nullptr;
    long long n_near = 0;
    for (int l = 0; l <= L && n > 0; ++l) {
      unsigned char* dec = static_cast<unsigned char*>(alloc(n));
      int* flags = static_cast<int*>(alloc(3 * n * sizeof(int)));
      int* pos = static_cast<int*>(alloc(3 * (n + 1) * sizeof(int)));
      k_decide<<<blocks(n), 256, 0, st>>>(n, fa, fb, dbox, ddiag, eta, l == L, dec, flags, flags + n, flags + 2 * n);
      IGB_PCUDA(cudaGetLastError());
      size_t tmp_bytes = 0;
      IGB_PCUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, flags, pos, static_cast<int>(n), st));
      void* tmp = alloc(tmp_bytes);
      int cnt[3];
      for (int k = 0; k < 3; ++k) {  // exclusive scans; count = last position + last flag
        IGB_PCUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, flags + k * n, pos + k * (n + 1), static_cast<int>(n), st));
        int last_pos = 0, last_flag = 0;
        IGB_PCUDA(cudaMemcpyAsync(&last_pos, pos + k * (n + 1) + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        IGB_PCUDA(cudaMemcpyAsync(&last_flag, flags + k * n + n - 1, sizeof(int), cudaMemcpyDeviceToHost, st));
        IGB_PCUDA(cudaStreamSynchronize(st));
        cnt[k] = last_pos + last_flag;
      }
      unsigned long long* fk = static_cast<unsigned long long*>(alloc(std::max(1, cnt[0]) * sizeof(unsigned long long)));
      if (cnt[1] > 0) near_keys = static_cast<unsigned long long*>(alloc(cnt[1] * sizeof(unsigned long long)));
      const long long nnext = 16LL * cnt[2];
      if (nnext > 0x7fffffffLL) throw std::runtime_error("B200 H2: too many block pairs for 32-bit indexing");
      int* na = static_cast<int*>(alloc(std::max<long long>(1, nnext) * sizeof(int)));
      int* nb = static_cast<int*>(alloc(std::max<long long>(1, nnext) * sizeof(int)));
      Level lv{P.npp, P.level_offset[l], l < L ? P.level_offset[l + 1] : 0, 1 << l};
      k_emit<<<blocks(n), 256, 0, st>>>(n, fa, fb, dec, pos, pos + (n + 1), pos + 2 * (n + 1), lv, epp, n1, fk, 0,
                                        near_keys, na, nb);
      IGB_PCUDA(cudaGetLastError());
      far_chunks.push_back(fk);
      far_counts.push_back(cnt[0]);
      if (cnt[1] > 0) n_near = cnt[1];
      fa = na;
      fb = nb;
      n = nnext;
    }
    // concatenate and sort the far keys; sort the near keys
    long long n_far = 0;
    for (long long c : far_counts) n_far += c;
    if (n_far > 0x7fffffffLL || n_near > 0x7fffffffLL)
      throw std::runtime_error("B200 H2: too many block pairs for 32-bit indexing");
    auto sort_keys = [&](unsigned long long* in, long long cnt) {
      unsigned long long* out = static_cast<unsigned long long*>(alloc(std::max<long long>(1, cnt) * 8));
      size_t tb = 0;
      IGB_PCUDA(cub::DeviceRadixSort::SortKeys(nullptr, tb, in, out, static_cast<int>(cnt), 0, 64, st));
      void* t = alloc(tb);
      IGB_PCUDA(cub::DeviceRadixSort::SortKeys(t, tb, in, out, static_cast<int>(cnt), 0, 64, st));
      return out;
    };
    unsigned long long* fall = static_cast<unsigned long long*>(alloc(std::max<long long>(1, n_far) * 8));
    {
      long long o = 0;
      for (size_t i = 0; i < far_chunks.size(); ++i) {
        if (far_counts[i])
          IGB_PCUDA(cudaMemcpyAsync(fall + o, far_chunks[i], far_counts[i] * 8, cudaMemcpyDeviceToDevice, st));
        o += far_counts[i];
      }
    }
    unsigned long long* fsorted = sort_keys(fall, n_far);
    unsigned long long* nsorted = n_near ? sort_keys(near_keys, n_near) : nullptr;
    // rows, columns, row starts, upper starts, transposes
    int* dfa = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dfb = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dtr = static_cast<int*>(alloc(std::max<long long>(1, n_far) * 4));
    int* dfrs = static_cast<int*>(alloc((nn + 1) * 4));
    int* dup = static_cast<int*>(alloc(nn * 4));
    int* dna = static_cast<int*>(alloc(std::max<long long>(1, n_near) * 4));
    int* dnb = static_cast<int*>(alloc(std::max<long long>(1, n_near) * 4));
    int* dnrs = static_cast<int*>(alloc((ne + 1) * 4));
    if (n_far) {
      k_split<<<blocks(n_far), 256, 0, st>>>(n_far, fsorted, dfa, dfb);
      k_trans<<<blocks(n_far), 256, 0, st>>>(n_far, fsorted, dtr);
    }
    k_rows<<<blocks(nn + 1), 256, 0, st>>>(nn, fsorted, n_far, dfrs, dup);
    if (n_near) k_split<<<blocks(n_near), 256, 0, st>>>(n_near, nsorted, dna, dnb);
    k_rows<<<blocks(ne + 1), 256, 0, st>>>(ne, nsorted, n_near, dnrs, nullptr);
    IGB_PCUDA(cudaGetLastError());
    P.far_a.resize(n_far);
    P.far_b.resize(n_far);
    P.far_trans.resize(n_far);
    P.far_row_start.resize(nn + 1);
    P.far_upper_start.resize(nn);
    P.near_a.resize(n_near);
    P.near_b.resize(n_near);
    P.near_row_start.resize(ne + 1);
    auto down = [&](std::vector<int>& v, const int* src) {
      if (!v.empty()) IGB_PCUDA(cudaMemcpyAsync(v.data(), src, v.size() * 4, cudaMemcpyDeviceToHost, st));
    };
    down(P.far_a, dfa);
    down(P.far_b, dfb);
    down(P.far_trans, dtr);
    down(P.far_row_start, dfrs);
    down(P.far_upper_start, dup);
    down(P.near_a, dna);
    down(P.near_b, dnb);
    down(P.near_row_start, dnrs);
    IGB_PCUDA(cudaStreamSynchronize(st));
  } catch (...) {
    release();
    throw;
  }
  release();
  for (int t : P.far_trans)
    if (t < 0) throw std::logic_error("B200 H2: admissible relation is not symmetric");
}

}  // namespace igb
