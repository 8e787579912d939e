// knn.cu -- exact top-K nearest means on the device (knn.py:33-75).
//
// Index: the snapshot of means is bucketed into a uniform grid (cell keys sorted
// with a device radix sort); each cell's means are contiguous (x, y, z, id).
// Query: points are processed in groups of G spatially-adjacent points (batch
// internal order, or Morton order for arbitrary query sets).  A group visits
// grid cells in Chebyshev rings around its own cell box; every thread keeps its
// point's kk = min(K+1, N) best (d2, id) in shared memory (d2 exactly as
// ((dx*dx + dy*dy) + dz*dz) in fp64, no FMA -- the cKDTree / numpy value).
// After ring r every unvisited mean is farther than r*h from every point of the
// group, so the group stops once all its threads hold kk candidates closer than
// that: the result is exact, ties included.
// Ordering (knn.py:58-74): rows by (sqrt(d2), id); a row whose K-th and
// (K+1)-th distances tie is resolved by (d2, id) over all means -- which is the
// kept (d2, id) order itself.
#include <cub/device/device_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "batch.cuh"

struct gsvr_knn_index {
  int64_t N = 0;
  double lo[3] = {0, 0, 0};
  double h = 1.0;
  int dims[3] = {1, 1, 1};
  int64_t ncells = 1;
  double4 *pts = nullptr;        // sorted by cell: (x, y, z, id)
  int32_t *cell_start = nullptr;  // ncells + 1
  cudaStream_t stream = nullptr;
  ~gsvr_knn_index() {
    if (pts) cudaFreeAsync(pts, stream);
    if (cell_start) cudaFreeAsync(cell_start, stream);
    cudaStreamSynchronize(stream);
  }
};

namespace gsvr {

struct GridView {
  double lo0, lo1, lo2, h;
  int d0, d1, d2;
  const double4 *pts;
  const int32_t *cell_start;
};

__device__ inline int cell_coord(double x, double lo, double h, int dim) {
  double f = floor((x - lo) / h);
  int c = f < 0.0 ? 0 : (f >= (double)dim ? dim - 1 : (int)f);
  return c;
}

__global__ void k_cell_keys(int64_t N, const double *__restrict__ m, GridView g, uint32_t *keys,
                            int32_t *vals, int *bad) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const double x = m[3 * i], y = m[3 * i + 1], z = m[3 * i + 2];
    if (!isfinite(x) || !isfinite(y) || !isfinite(z)) atomicExch(bad, 1);
    const int cx = cell_coord(x, g.lo0, g.h, g.d0), cy = cell_coord(y, g.lo1, g.h, g.d1),
              cz = cell_coord(z, g.lo2, g.h, g.d2);
    keys[i] = (uint32_t)(((int64_t)cz * g.d1 + cy) * g.d0 + cx);
    vals[i] = (int32_t)i;
  }
}

__global__ void k_cell_fill(int64_t N, const double *__restrict__ m, const int32_t *__restrict__ order,
                            double4 *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = order[i];
    out[i] = make_double4(m[3 * j], m[3 * j + 1], m[3 * j + 2], (double)j);
  }
}

__global__ void k_cell_start(int64_t ncells, int64_t N, const uint32_t *__restrict__ skeys, int32_t *start) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c <= ncells; c += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = N;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)skeys[mid] < c) lo = mid + 1; else hi = mid;
    }
    start[c] = (int32_t)lo;
  }
}

struct QuerySrc {
  const double *pts;     // (M,3) query points, or null -> batch mode
  const double *x0s;     // batch mode: nominal points, internal order
  const int32_t *sid;    // batch mode: slice ids
  const double *Rc, *tv; // batch mode: per-slice corrections
  const int32_t *orow;   // output row per query position (null -> identity)
  int64_t M;
};

__device__ inline void query_point(const QuerySrc &q, int64_t i, double x[3]) {
  if (q.pts) {
    x[0] = q.pts[3 * i]; x[1] = q.pts[3 * i + 1]; x[2] = q.pts[3 * i + 2];
  } else {
    // train.py:305-309 einsum order: ((R0 a0 + R1 a1) + R2 a2) + t
    const int s = q.sid[i];
    const double a0 = q.x0s[3 * i], a1 = q.x0s[3 * i + 1], a2 = q.x0s[3 * i + 2];
    for (int r = 0; r < 3; ++r) {
      const double *R = q.Rc + 9 * s + 3 * r;
      x[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[0], a0), __dmul_rn(R[1], a1)), __dmul_rn(R[2], a2)),
                       q.tv[3 * s + r]);
    }
  }
}

template <int G>
__global__ void __launch_bounds__(G) k_knn_query(QuerySrc q, GridView g, int K, int kk, void *out, int out_i64) {
  extern __shared__ unsigned char sm_raw[];
  double *sd = reinterpret_cast<double *>(sm_raw);             // [kk][G]
  int32_t *si = reinterpret_cast<int32_t *>(sd + (size_t)kk * G);  // [kk][G]
  __shared__ int box[6];
  const int tid = threadIdx.x;
  const int64_t i = (int64_t)blockIdx.x * G + tid;
  const bool active = i < q.M;
  double x[3] = {0, 0, 0};
  if (active) query_point(q, i, x);
  // group cell box
  int c[3] = {0, 0, 0};
  if (active) {
    c[0] = cell_coord(x[0], g.lo0, g.h, g.d0);
    c[1] = cell_coord(x[1], g.lo1, g.h, g.d1);
    c[2] = cell_coord(x[2], g.lo2, g.h, g.d2);
  }
  if (tid == 0) {
    box[0] = box[1] = box[2] = INT32_MAX;
    box[3] = box[4] = box[5] = -1;
  }
  __syncthreads();
  if (active) {
    for (int d = 0; d < 3; ++d) {
      atomicMin(&box[d], c[d]);
      atomicMax(&box[3 + d], c[d]);
    }
  }
  __syncthreads();
  const int glo[3] = {box[0], box[1], box[2]}, ghi[3] = {box[3], box[4], box[5]};
  const int dims[3] = {g.d0, g.d1, g.d2};

  int count = 0;
  double worst = INFINITY;
  int worst_id = INT32_MAX;
  auto consider = [&](const double4 cand) {
    const double dx = __dsub_rn(x[0], cand.x), dy = __dsub_rn(x[1], cand.y), dz = __dsub_rn(x[2], cand.z);
    const double d2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
    const int id = (int)cand.w;
    if (count == kk && !(d2 < worst || (d2 == worst && id < worst_id))) return;
    int pos = count < kk ? count++ : kk - 1;
    while (pos > 0) {
      const double pd = sd[(pos - 1) * G + tid];
      const int pi = si[(pos - 1) * G + tid];
      if (pd < d2 || (pd == d2 && pi < id)) break;
      sd[pos * G + tid] = pd;
      si[pos * G + tid] = pi;
      --pos;
    }
    sd[pos * G + tid] = d2;
    si[pos * G + tid] = id;
    if (count == kk) {
      worst = sd[(kk - 1) * G + tid];
      worst_id = si[(kk - 1) * G + tid];
    }
  };
  auto scan_range = [&](int64_t a, int64_t b) {
    for (int64_t e = a; e < b; ++e) {
      const double4 cand = g.pts[e];
      if (active) consider(cand);
    }
  };

  for (int r = 0;; ++r) {
    int lo[3], hi[3];
    bool full = true;
    for (int d = 0; d < 3; ++d) {
      lo[d] = glo[d] - r;
      hi[d] = ghi[d] + r;
      full = full && lo[d] <= 0 && hi[d] >= dims[d] - 1;
    }
    const int zlo = max(lo[2], 0), zhi = min(hi[2], dims[2] - 1);
    const int ylo = max(lo[1], 0), yhi = min(hi[1], dims[1] - 1);
    const int xlo = max(lo[0], 0), xhi = min(hi[0], dims[0] - 1);
    for (int z = zlo; z <= zhi; ++z) {
      for (int y = ylo; y <= yhi; ++y) {
        const int64_t row = ((int64_t)z * dims[1] + y) * dims[0];
        const bool shell = r == 0 || z == lo[2] || z == hi[2] || y == lo[1] || y == hi[1];
        if (shell) {
          scan_range(g.cell_start[row + xlo], g.cell_start[row + xhi + 1]);
        } else {
          if (lo[0] >= 0) scan_range(g.cell_start[row + lo[0]], g.cell_start[row + lo[0] + 1]);
          if (hi[0] <= dims[0] - 1) scan_range(g.cell_start[row + hi[0]], g.cell_start[row + hi[0] + 1]);
        }
      }
    }
    const double gap = (double)r * g.h * (1.0 - 1e-9);
    const bool done = !active || full || (count == kk && worst < gap * gap);
    if (__syncthreads_and(done)) break;
  }
  if (!active) return;
  GSVR_DCHECK(count == kk, "knn count", count, kk);

  // knn.py:58-74 ordering
  const bool tie = kk > K && sqrt(sd[(K - 1) * G + tid]) == sqrt(sd[K * G + tid]);
  if (!tie) {
    int a = 0;
    while (a < K) {
      const double da = sqrt(sd[a * G + tid]);
      int b = a + 1;
      while (b < kk && sqrt(sd[b * G + tid]) == da) ++b;
      for (int u = a + 1; u < b; ++u) {  // insertion sort of the run by id
        const int id = si[u * G + tid];
        const double dv = sd[u * G + tid];
        int v = u;
        while (v > a && si[(v - 1) * G + tid] > id) {
          si[v * G + tid] = si[(v - 1) * G + tid];
          sd[v * G + tid] = sd[(v - 1) * G + tid];
          --v;
        }
        si[v * G + tid] = id;
        sd[v * G + tid] = dv;
      }
      a = b;
    }
  }
  const int64_t row = q.orow ? (int64_t)q.orow[i] : i;
  if (out_i64) {
    int64_t *o = reinterpret_cast<int64_t *>(out) + row * K;
    for (int k = 0; k < K; ++k) o[k] = si[k * G + tid];
  } else {
    int32_t *o = reinterpret_cast<int32_t *>(out) + row * K;
    for (int k = 0; k < K; ++k) o[k] = si[k * G + tid];
  }
}

int knn_run(const gsvr_knn_index *ix, const QuerySrc &q, int64_t K, void *out, int out_i64, cudaStream_t st) {
  if (K < 1 || K > ix->N) return fail(GSVR_ERR_INVALID, "K must be in [1, %lld], got %lld", (long long)ix->N,
                                      (long long)K);
  if (q.M == 0) return GSVR_OK;
  const int kk = (int)std::min<int64_t>(K + 1, ix->N);
  GridView g{ix->lo[0], ix->lo[1], ix->lo[2], ix->h, ix->dims[0], ix->dims[1], ix->dims[2], ix->pts,
             ix->cell_start};
  const size_t per = (size_t)kk * 12;
  const size_t limit = 200 * 1024;
#define GSVR_KNN(GSZ)                                                                                      \
  do {                                                                                                     \
    const size_t sm = per * GSZ;                                                                           \
    GSVR_CUDA(cudaFuncSetAttribute(k_knn_query<GSZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm)); \
    k_knn_query<GSZ><<<(unsigned)((q.M + GSZ - 1) / GSZ), GSZ, sm, st>>>(q, g, (int)K, kk, out, out_i64);   \
    GSVR_LAUNCH_CHECK("k_knn_query");                                                                      \
    return GSVR_OK;                                                                                        \
  } while (0)
  if (per * 128 <= limit) GSVR_KNN(128);
  if (per * 64 <= limit) GSVR_KNN(64);
  if (per * 32 <= limit) GSVR_KNN(32);
#undef GSVR_KNN
  return fail(GSVR_ERR_INVALID, "K=%lld too large for the device K-NN", (long long)K);
}

__global__ void k_morton_points(int64_t M, const double *__restrict__ p, double3 lo, double3 inv,
                                unsigned long long *keys, int32_t *vals) {
  const unsigned long long qmax = (1ull << 21) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    double f[3] = {(p[3 * i] - lo.x) * inv.x, (p[3 * i + 1] - lo.y) * inv.y, (p[3 * i + 2] - lo.z) * inv.z};
    unsigned long long code = 0;
    for (int d = 0; d < 3; ++d) {
      double qv = f[d] * (double)qmax;
      unsigned long long u = qv <= 0.0 ? 0ull : (qv >= (double)qmax ? qmax : (unsigned long long)qv);
      code |= spread3(u) << (2 - d);
    }
    keys[i] = code;
    vals[i] = (int32_t)i;
  }
}

__global__ void k_gather_points(int64_t M, const double *__restrict__ p, const int32_t *__restrict__ order,
                                double *__restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < M; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = order[i];
    out[3 * i] = p[3 * j];
    out[3 * i + 1] = p[3 * j + 1];
    out[3 * i + 2] = p[3 * j + 2];
  }
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_knn_build(int64_t N, const double *means, gsvr_knn_index **out, void *stream) {
  *out = nullptr;
  if (N < 1) return fail(GSVR_ERR_INVALID, "means must be a non-empty (N, 3) array");
  if (N > INT32_MAX) return fail(GSVR_ERR_INVALID, "too many means");
  cudaStream_t st = as_stream(stream);
  Scratch bbk;
  GSVR_TRY(bbk.alloc(48, st));
  double bb[6];
  if (bbox3(means, N, bbk.as<unsigned long long>(), bb, st) != GSVR_OK)
    return fail(GSVR_ERR_INVALID, "non-finite means");
  auto *ix = new gsvr_knn_index();
  ix->N = N;
  ix->stream = st;
  double ext[3];
  double emax = 0.0;
  for (int d = 0; d < 3; ++d) {
    ix->lo[d] = bb[d];
    ext[d] = bb[3 + d] - bb[d];
    emax = std::max(emax, ext[d]);
  }
  // ~3 means per occupied cell volume; degenerate extents get one cell
  double vol = 1.0;
  int nd = 0;
  for (int d = 0; d < 3; ++d)
    if (ext[d] > emax * 1e-6 && ext[d] > 0) vol *= ext[d], ++nd;
  double h = emax > 0 ? std::pow(vol * 3.0 / (double)N, 1.0 / std::max(nd, 1)) : 1.0;
  if (!(h > 0) || !std::isfinite(h)) h = emax > 0 ? emax : 1.0;
  for (;;) {
    int64_t nc = 1;
    for (int d = 0; d < 3; ++d) {
      ix->dims[d] = (int)std::min<double>(std::floor(ext[d] / h) + 1, 1 << 20);
      nc *= ix->dims[d];
    }
    if (nc <= std::max<int64_t>(4 * N, 64) && nc < (1ll << 30)) {
      ix->ncells = nc;
      break;
    }
    h *= 1.25;
  }
  ix->h = h;
  GridView g{ix->lo[0], ix->lo[1], ix->lo[2], h, ix->dims[0], ix->dims[1], ix->dims[2], nullptr, nullptr};
  Scratch keys, keys2, vals, vals2, tmp, flag;
  auto bail = [&](int rc) { delete ix; return rc; };
  if (int rc = keys.alloc(N * 4, st)) return bail(rc);
  if (int rc = keys2.alloc(N * 4, st)) return bail(rc);
  if (int rc = vals.alloc(N * 4, st)) return bail(rc);
  if (int rc = vals2.alloc(N * 4, st)) return bail(rc);
  if (int rc = flag.alloc(4, st)) return bail(rc);
  cudaMemsetAsync(flag.ptr, 0, 4, st);
  k_cell_keys<<<grid_for(N, 256), 256, 0, st>>>(N, means, g, keys.as<uint32_t>(), vals.as<int32_t>(), flag.as<int>());
  int bits = 1;
  while ((1ll << bits) < ix->ncells) ++bits;
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(), vals.as<int32_t>(),
                                  vals2.as<int32_t>(), (int)N, 0, bits, st);
  if (int rc = tmp.alloc(tb, st)) return bail(rc);
  cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, keys.as<uint32_t>(), keys2.as<uint32_t>(), vals.as<int32_t>(),
                                  vals2.as<int32_t>(), (int)N, 0, bits, st);
  if (cudaMallocAsync((void **)&ix->pts, N * 32, st) != cudaSuccess ||
      cudaMallocAsync((void **)&ix->cell_start, (ix->ncells + 1) * 4, st) != cudaSuccess)
    return bail(fail(GSVR_ERR_CUDA, "out of device memory for the K-NN index"));
  k_cell_fill<<<grid_for(N, 256), 256, 0, st>>>(N, means, vals2.as<int32_t>(), ix->pts);
  k_cell_start<<<grid_for(ix->ncells + 1, 256), 256, 0, st>>>(ix->ncells, N, keys2.as<uint32_t>(), ix->cell_start);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return bail(cuda_status(e, "knn build"));
  int bad = 0;
  cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return bail(cuda_status(cudaGetLastError(), "knn build"));
  if (bad) return bail(fail(GSVR_ERR_INVALID, "non-finite means"));
  *out = ix;
  return GSVR_OK;
}

void gsvr_knn_free(gsvr_knn_index *index) { delete index; }
int64_t gsvr_knn_count(const gsvr_knn_index *index) { return index ? index->N : 0; }

int gsvr_knn_query(const gsvr_knn_index *ix, int64_t M, const double *points, int64_t K, void *out, int out_i64,
                   void *stream) {
  cudaStream_t st = as_stream(stream);
  if (K < 1 || K > ix->N) return fail(GSVR_ERR_INVALID, "K must be in [1, %lld], got %lld", (long long)ix->N,
                                      (long long)K);
  if (M == 0) return GSVR_OK;
  // Morton-order the queries so each group of G is spatially compact.
  Scratch bbk, keys, keys2, vals, order, tmp, sorted;
  GSVR_TRY(bbk.alloc(48, st));
  double bb[6];
  if (bbox3(points, M, bbk.as<unsigned long long>(), bb, st) != GSVR_OK)
    return fail(GSVR_ERR_INVALID, "non-finite query points");
  double3 lo = make_double3(bb[0], bb[1], bb[2]);
  double e0 = bb[3] - bb[0], e1 = bb[4] - bb[1], e2 = bb[5] - bb[2];
  double3 inv = make_double3(e0 > 0 ? 1 / e0 : 0, e1 > 0 ? 1 / e1 : 0, e2 > 0 ? 1 / e2 : 0);
  GSVR_TRY(keys.alloc(M * 8, st));
  GSVR_TRY(keys2.alloc(M * 8, st));
  GSVR_TRY(vals.alloc(M * 4, st));
  GSVR_TRY(order.alloc(M * 4, st));
  GSVR_TRY(sorted.alloc(M * 24, st));
  k_morton_points<<<grid_for(M, 256), 256, 0, st>>>(M, points, lo, inv, keys.as<unsigned long long>(),
                                                    vals.as<int32_t>());
  size_t tb = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tb, keys.as<unsigned long long>(), keys2.as<unsigned long long>(),
                                  vals.as<int32_t>(), order.as<int32_t>(), (int)M, 0, 63, st);
  GSVR_TRY(tmp.alloc(tb, st));
  cub::DeviceRadixSort::SortPairs(tmp.ptr, tb, keys.as<unsigned long long>(), keys2.as<unsigned long long>(),
                                  vals.as<int32_t>(), order.as<int32_t>(), (int)M, 0, 63, st);
  k_gather_points<<<grid_for(M, 256), 256, 0, st>>>(M, points, order.as<int32_t>(), sorted.as<double>());
  GSVR_LAUNCH_CHECK("knn query prep");
  QuerySrc q{sorted.as<double>(), nullptr, nullptr, nullptr, nullptr, order.as<int32_t>(), M};
  return knn_run(ix, q, K, out, out_i64, st);
}

int gsvr_batch_refresh(gsvr_batch *b, const gsvr_knn_index *ix, int64_t K, const double *Rc, const double *tvec,
                       void *stream) {
  cudaStream_t st = as_stream(stream);
  if (b->nbr_int && b->K != K) b->release_binning();
  if (!b->nbr_int) GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_int, b->P * K * 4, st));
  QuerySrc q{nullptr, b->x0s, b->sid_s, Rc, tvec, nullptr, b->P};
  GSVR_TRY(knn_run(ix, q, K, b->nbr_int, 0, st));
  return batch_bin_internal(b, K, ix->N, st);
}

}  // extern "C"
