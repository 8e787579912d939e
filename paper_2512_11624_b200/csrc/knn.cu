// knn.cu -- exact top-K nearest means on the device (knn.py:33-75).
//
// Index: the snapshot of means is bucketed into a uniform grid (cell keys sorted
// with a device radix sort); each cell's means are contiguous (x, y, z, id).
// Query: one query per thread; each warp is a group of 32 spatially-adjacent
// points (batch internal order, or Morton order for arbitrary query sets) that
// visits grid cells in Chebyshev rings around its own cell box.  Every thread
// keeps its point's kk = min(K+1, N) best (d2, id) in a shared-memory max-heap
// (d2 exactly as ((dx*dx + dy*dy) + dz*dz) in fp64, no FMA -- the cKDTree /
// numpy value).  Cell rows farther than every lane's current kk-th distance are
// skipped; after ring r every unvisited mean is farther than r*h from every
// point of the warp, so the warp stops once all its lanes hold kk candidates
// closer than that: the result is exact, ties included.
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
  double *means = nullptr;       // (N, 3) by id (refresh seeds)
  int32_t *cell_start = nullptr;  // ncells + 1
  cudaStream_t stream = nullptr;
  ~gsvr_knn_index() {
    if (pts) cudaFreeAsync(pts, stream);
    if (means) cudaFreeAsync(means, stream);
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
  // refresh seeds (batch mode, optional): K ids per row + the (K+1)-th; any kk
  // distinct means bound the kk-th distance from above
  const int32_t *seed;
  const int32_t *seed_next;
  const double *means;  // (N, 3) by id
  int32_t *out_next;    // (K+1)-th id of every row (or null)
  const int32_t *rows = nullptr;  // batch mode: query positions -> batch rows (fallback lists), or null
  int one_per_warp = 0;           // rows list: one row per warp (scattered rows: no shared warp box)
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

// Query position in grid-cell units (fp32) for row pruning: a conservative
// lower bound of the squared distance (in cells^2) from the query to the cell
// box [a0, b0] x {y} x {z}.  The position is clamped into the grid box
// [0, dims]: a boundary cell (which extends to infinity like the clamped
// cell_coord) then gets gap 0 to any point beyond it, and every other gap can
// only shrink -- still a lower bound, with no per-axis boundary selects.  fp32
// with a 1e-3-cell shrink instead of fp64 (the coordinate rounding is < 1e-4
// cells): pruning only ever keeps extra rows.
struct CellPos {
  float c[3];
  __device__ void init(const double x[3], const GridView &g) {
    const double cc[3] = {(x[0] - g.lo0) / g.h, (x[1] - g.lo1) / g.h, (x[2] - g.lo2) / g.h};
    const int dims[3] = {g.d0, g.d1, g.d2};
    for (int d = 0; d < 3; ++d) c[d] = (float)fmin(fmax(cc[d], 0.0), (double)dims[d]);
  }
  __device__ float box_d2(int a0, int b0, int y, int z, const int dims[3]) const {
    (void)dims;
    const float lo3[3] = {(float)a0 - 1e-3f, (float)y - 1e-3f, (float)z - 1e-3f};
    const float hi3[3] = {(float)(b0 + 1) + 1e-3f, (float)(y + 1) + 1e-3f, (float)(z + 1) + 1e-3f};
    float s = 0.f;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const float gap = fmaxf(fmaxf(lo3[d] - c[d], c[d] - hi3[d]), 0.f);
      s = fmaf(gap, gap, s);
    }
    return s;
  }
};
// an fp32 upper bound of d2 / h^2 (cells^2) for comparisons with box_d2
__device__ inline float cells2_bound(double d2, double inv_h2) {
  if (!(d2 >= 0.0)) return -1.f;
  return (float)(d2 * inv_h2) * (1.0f + 1e-5f) + 1e-6f;
}

// Per-thread bounded max-heap of the kk best (d2, id) so far, in shared memory
// (column layout [slot][G]: lanes never conflict).  Order is (d2, id)
// lexicographic, so the kept set is exactly the sorted-insertion set.
struct KnnHeap {
  double *d;
  int32_t *id;
  int G;
  __device__ double &D(int k) const { return d[k * G]; }
  __device__ int32_t &I(int k) const { return id[k * G]; }
};

__device__ inline bool knn_less(double da, int ia, double db, int ib) { return da < db || (da == db && ia < ib); }

// sift the (dv, iv) hole at 'pos' down inside heap[0, n)
__device__ inline void knn_sift_down(const KnnHeap &h, int pos, int n, double dv, int iv) {
  for (;;) {
    int c = 2 * pos + 1;
    if (c >= n) break;
    double dc = h.D(c);
    int ic = h.I(c);
    if (c + 1 < n) {
      const double d1 = h.D(c + 1);
      const int i1 = h.I(c + 1);
      if (knn_less(dc, ic, d1, i1)) dc = d1, ic = i1, ++c;
    }
    if (!knn_less(dv, iv, dc, ic)) break;
    h.D(pos) = dc;
    h.I(pos) = ic;
    pos = c;
  }
  h.D(pos) = dv;
  h.I(pos) = iv;
}

// Exact K-NN of one query per thread; each WARP is an independent group of 32
// spatially-adjacent queries scanning Chebyshev cell rings around its own cell
// box.  Cell rows whose box is farther from every lane's point than that
// lane's current kk-th distance are skipped (warp vote), and after ring r every
// unvisited mean is farther than r*h from every point of the warp, so the warp
// stops once all its lanes hold kk candidates closer than that.
#ifdef GSVR_KNN_STATS
// diagnostics build only: [0] warps [1] candidates scanned per warp [2] rows
// scanned [3] rows skipped [4] sift-ups [5] sift-downs [6] rings [7] lane
// candidates under the bound
__device__ unsigned long long g_knn_stats[8];
#define KNN_STAT(i, v) atomicAdd(&g_knn_stats[i], (unsigned long long)(v))
#else
#define KNN_STAT(i, v) ((void)0)
#endif
#ifndef GSVR_KNN_UNROLL
#define GSVR_KNN_UNROLL 4
#endif
template <int G>
__global__ void __launch_bounds__(G) k_knn_query(QuerySrc q, GridView g, int K, int kk, void *out, int out_i64) {
  extern __shared__ unsigned char sm_raw[];
  const int tid = threadIdx.x, lane = tid & 31;
  KnnHeap hp{reinterpret_cast<double *>(sm_raw) + tid,
             reinterpret_cast<int32_t *>(reinterpret_cast<double *>(sm_raw) + (size_t)kk * G) + tid, G};
  const int64_t pos = q.one_per_warp ? (int64_t)blockIdx.x : (int64_t)blockIdx.x * G + tid;
  const bool active = pos < q.M && (!q.one_per_warp || tid == 0);
  const int64_t i = (q.rows && active) ? (int64_t)q.rows[pos] : pos;
  double x[3] = {0, 0, 0};
  if (active) query_point(q, i, x);
  const int dims[3] = {g.d0, g.d1, g.d2};
  const double glo[3] = {g.lo0, g.lo1, g.lo2};
  int c[3];
  c[0] = cell_coord(x[0], g.lo0, g.h, g.d0);
  c[1] = cell_coord(x[1], g.lo1, g.h, g.d1);
  c[2] = cell_coord(x[2], g.lo2, g.h, g.d2);
  int blo[3], bhi[3];
  for (int d = 0; d < 3; ++d) {
    blo[d] = __reduce_min_sync(0xffffffffu, active ? c[d] : INT32_MAX);
    bhi[d] = __reduce_max_sync(0xffffffffu, active ? c[d] : -1);
  }
  if (bhi[0] < 0) return;  // whole warp past the end
  if (lane == 0) KNN_STAT(0, 1);

  auto dist2 = [&](double mx, double my, double mz) {
    const double dx = __dsub_rn(x[0], mx), dy = __dsub_rn(x[1], my), dz = __dsub_rn(x[2], mz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  };
  // seed bound T >= this point's kk-th smallest d2 (+inf without seeds)
  double T = INFINITY;
  if (q.seed && active) {
    const int32_t *sr = q.seed + i * K;
    double t = 0.0;
    for (int k = 0; k < kk; ++k) {
      const int j = k < K ? sr[k] : q.seed_next[i];
      t = fmax(t, dist2(q.means[3 * j], q.means[3 * j + 1], q.means[3 * j + 2]));
    }
    T = t;
  }

  int count = 0;
  double worst = INFINITY;
  int worst_id = INT32_MAX;
  CellPos cp;
  cp.init(x, g);
  const double inv_h2 = 1.0 / (g.h * g.h);
  (void)glo;
  auto consider = [&](const double d2, const int id) {
    if (d2 > T) return;  // at least kk means are at d2 <= T
    if (count < kk) {  // sift up
      KNN_STAT(4, 1);
      int pos = count++;
      while (pos > 0) {
        const int par = (pos - 1) >> 1;
        const double pd = hp.D(par);
        const int pi = hp.I(par);
        if (!knn_less(pd, pi, d2, id)) break;
        hp.D(pos) = pd;
        hp.I(pos) = pi;
        pos = par;
      }
      hp.D(pos) = d2;
      hp.I(pos) = id;
      if (count == kk) worst = hp.D(0), worst_id = hp.I(0);
    } else if (knn_less(d2, id, worst, worst_id)) {
      KNN_STAT(5, 1);
      knn_sift_down(hp, 0, kk, d2, id);
      worst = hp.D(0);
      worst_id = hp.I(0);
    }
  };
  // candidates [e0, e1) of cells a0..b0 of row (y, z)
  auto scan_cells = [&](int a0, int b0, int y, int z, int e0, int e1) {
    const bool need = active && cp.box_d2(a0, b0, y, z, dims) <= cells2_bound(count < kk ? T : worst, inv_h2);
    if (!__any_sync(0xffffffffu, need)) {
      if (lane == 0) KNN_STAT(3, 1);
      return;
    }
    if (lane == 0) KNN_STAT(2, 1), KNN_STAT(1, e1 - e0);
    int e = e0;
    // KU candidates per step: independent loads and fp64 distance chains (ILP);
    // only those under the current bound reach the (single) heap update
    constexpr int KU = GSVR_KNN_UNROLL;
    for (; e + KU <= e1; e += KU) {
      double4 c4[KU];
#pragma unroll
      for (int u = 0; u < KU; ++u) c4[u] = g.pts[e + u];
      double d4[KU];
      unsigned m = 0;
      const double bnd = count < kk ? T : worst;
#pragma unroll
      for (int u = 0; u < KU; ++u) {
        d4[u] = dist2(c4[u].x, c4[u].y, c4[u].z);
        m |= (need && d4[u] <= bnd) ? 1u << u : 0u;
#ifdef GSVR_KNN_STATS
        if (need && d4[u] <= bnd) KNN_STAT(7, 1);
#endif
      }
      while (m) {
        const int u = __ffs(m) - 1;
        m &= m - 1;
        double du = d4[0];
        int iu = (int)c4[0].w;
#pragma unroll
        for (int v = 1; v < KU; ++v)
          if (u == v) du = d4[v], iu = (int)c4[v].w;
        consider(du, iu);
      }
    }
    for (; e < e1; ++e) {
      const double4 cand = g.pts[e];
      if (need) consider(dist2(cand.x, cand.y, cand.z), (int)cand.w);
    }
  };

  for (int r = 0;; ++r) {
    int lo[3], hi[3];
    bool full = true;
    for (int d = 0; d < 3; ++d) {
      lo[d] = blo[d] - r;
      hi[d] = bhi[d] + r;
      full = full && lo[d] <= 0 && hi[d] >= dims[d] - 1;
    }
    const int zlo = max(lo[2], 0), zhi = min(hi[2], dims[2] - 1);
    const int ylo = max(lo[1], 0), yhi = min(hi[1], dims[1] - 1);
    const int xlo = max(lo[0], 0), xhi = min(hi[0], dims[0] - 1);
    // the ring's row segments (shell rows: the whole x range; interior rows:
    // the two end cells) in slots 2*row + side; each batch of 32 slots has its
    // cell_start bounds loaded by the lanes in parallel, then the warp walks
    // them in order (one load latency per 32 rows instead of one per row)
    const int ny = yhi - ylo + 1, nslots = 2 * ny * (zhi - zlo + 1);
    for (int sb = 0; sb < nslots; sb += 32) {
      const int sl = sb + lane;
      int sa = 1, sbx = 0, sy = 0, sz = 0, se0 = 0, se1 = 0;
      if (sl < nslots) {
        const int ri = sl >> 1, side = sl & 1;
        sz = zlo + ri / ny;
        sy = ylo + ri - (ri / ny) * ny;
        const bool shell = r == 0 || sz == lo[2] || sz == hi[2] || sy == lo[1] || sy == hi[1];
        if (shell) {
          if (side == 0) sa = xlo, sbx = xhi;
        } else if (side == 0) {
          if (lo[0] >= 0) sa = sbx = lo[0];
        } else if (hi[0] <= dims[0] - 1) {
          sa = sbx = hi[0];
        }
        if (sa <= sbx) {
          const int64_t row = ((int64_t)sz * dims[1] + sy) * dims[0];
          se0 = g.cell_start[row + sa];
          se1 = g.cell_start[row + sbx + 1];
        }
      }
      const int cnt = min(32, nslots - sb);
      for (int j = 0; j < cnt; ++j) {
        const int e0 = __shfl_sync(0xffffffffu, se0, j), e1 = __shfl_sync(0xffffffffu, se1, j);
        if (e0 >= e1) continue;  // no means in the segment (or an empty slot)
        scan_cells(__shfl_sync(0xffffffffu, sa, j), __shfl_sync(0xffffffffu, sbx, j),
                   __shfl_sync(0xffffffffu, sy, j), __shfl_sync(0xffffffffu, sz, j), e0, e1);
      }
    }
    if (lane == 0) KNN_STAT(6, 1);
    const double gap = (double)r * g.h * (1.0 - 1e-9);
    const bool done = !active || full || (count == kk && worst < gap * gap);
    if (__all_sync(0xffffffffu, done)) break;
  }
  if (!active) return;
  GSVR_DCHECK(count == kk, "knn count", count, kk);
  // heap sort in place -> ascending (d2, id)
  for (int n = kk - 1; n > 0; --n) {
    const double dv = hp.D(n);
    const int iv = hp.I(n);
    hp.D(n) = hp.D(0);
    hp.I(n) = hp.I(0);
    knn_sift_down(hp, 0, n, dv, iv);
  }
  const double *sd = hp.d;
  const int32_t *si = hp.id;
  if (q.out_next) q.out_next[i] = kk > K ? si[K * G] : -1;

  // knn.py:58-74 ordering.  sqrt(lo) == sqrt(hi) for lo <= hi (adjacent kept
  // entries); sqrt only when the values are within 1e-14 relative (beyond
  // that the square roots are > 20 ulp apart).
  auto same_dist = [](double lo, double hi) {
    if (hi == lo) return true;
    if (hi > lo * (1.0 + 1e-14)) return false;
    return sqrt(lo) == sqrt(hi);
  };
  const bool tie = kk > K && same_dist(sd[(K - 1) * G], sd[K * G]);
  if (!tie) {
    int a = 0;
    while (a < K) {
      int b = a + 1;
      while (b < kk && same_dist(sd[(b - 1) * G], sd[b * G])) ++b;  // equal-sqrt run [a, b)
      for (int u = a + 1; u < b; ++u) {  // insertion sort of the run by id
        const int id = hp.I(u);
        const double dv = hp.D(u);
        int v = u;
        while (v > a && hp.I(v - 1) > id) {
          hp.I(v) = hp.I(v - 1);
          hp.D(v) = hp.D(v - 1);
          --v;
        }
        hp.I(v) = id;
        hp.D(v) = dv;
      }
      a = b;
    }
  }
  const int64_t row = q.orow ? (int64_t)q.orow[i] : i;
  if (out_i64) {
    int64_t *o = reinterpret_cast<int64_t *>(out) + row * K;
    for (int k = 0; k < K; ++k) o[k] = si[k * G];
  } else {
    int32_t *o = reinterpret_cast<int32_t *>(out) + row * K;
    for (int k = 0; k < K; ++k) o[k] = si[k * G];
  }
}

// ---------------------------------------------------------------------------
// Seeded refresh without heaps: two-pass distance-histogram selection.
//
// A refresh inside a fit has the previous lists of every row (K ids + the
// (K+1)-th): their kk distinct means bound the new kk-th distance by
// T = max of their d2 under the moved points (the heap kernel's seed bound).
// Pass 1 scans the cells (same warp-group ring scan as k_knn_query) and
// histograms every candidate with d2 <= T into kSelBins bins over [0, T]
// (per-lane u16 counters in shared memory); the bin b* where the cumulative
// count reaches kk splits the candidates: bins < b* are certainly in, bin b*
// holds the boundary.  Pass 2 rescans the cells (tighter bound: bin <= b*) and
// writes every bin < b* entry straight to its bin's slot range of the output
// row (ids) and a d2 scratch row, and the b* entries to a small per-lane list;
// the boundary list is sorted and its first kk - c_lo entries complete the
// row.  A final insertion sort only reorders inside bins, and the
// knn.py:58-74 ordering rules run on the sorted row exactly as in the heap
// kernel.  No per-candidate heap operation: shared memory per query is 128 B
// of counters + the boundary list (vs 612 B of heap), so 4x more warps stay
// resident.  Rows whose boundary bin holds more than kSelCap entries (exact
// distance ties en masse) are handed to the heap kernel (fallback list).
#ifndef GSVR_SEL_CAP
#define GSVR_SEL_CAP 12
#endif
#ifndef GSVR_SEL_UNROLL
#define GSVR_SEL_UNROLL 2
#endif
#ifndef GSVR_SEL_MINB
#define GSVR_SEL_MINB 7
#endif
constexpr int kSelBins = 64;
constexpr int kSelCap = GSVR_SEL_CAP;
constexpr int kSelWarps = 4;

template <int WPB>
__global__ void __launch_bounds__(32 * WPB, GSVR_SEL_MINB) k_knn_select(QuerySrc q, GridView g, int K, int kk, int32_t *out,
                                                         double *scr, int64_t row0, int32_t *fb_rows,
                                                         int *fb_count) {
  __shared__ uint8_t s_hist[WPB][kSelBins][32];  // per-lane bin counters (saturation -> heap kernel)
  __shared__ double s_bd[WPB][kSelCap][32];
  __shared__ int32_t s_bi[WPB][kSelCap][32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t i = row0 + ((int64_t)blockIdx.x * WPB + warp) * 32 + lane;  // rows [row0, q.M) of this launch
  bool active = i < q.M;
  double x[3] = {0, 0, 0};
  if (active) query_point(q, i, x);
  const int dims[3] = {g.d0, g.d1, g.d2};
  const double glo[3] = {g.lo0, g.lo1, g.lo2};
  int c[3];
  c[0] = cell_coord(x[0], g.lo0, g.h, g.d0);
  c[1] = cell_coord(x[1], g.lo1, g.h, g.d1);
  c[2] = cell_coord(x[2], g.lo2, g.h, g.d2);
  int blo[3], bhi[3];
  for (int d = 0; d < 3; ++d) {
    blo[d] = __reduce_min_sync(0xffffffffu, active ? c[d] : INT32_MAX);
    bhi[d] = __reduce_max_sync(0xffffffffu, active ? c[d] : -1);
  }
  if (bhi[0] < 0) return;  // whole warp past the end
  auto dist2 = [&](double mx, double my, double mz) {
    const double dx = __dsub_rn(x[0], mx), dy = __dsub_rn(x[1], my), dz = __dsub_rn(x[2], mz);
    return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
  };
  double T = -1.0;  // seed bound (>= the kk-th smallest d2)
  if (active) {
    const int32_t *sr = q.seed + i * K;
    double t = 0.0;
    for (int k = 0; k < kk; ++k) {
      const int j = k < K ? sr[k] : q.seed_next[i];
      t = fmax(t, dist2(q.means[3 * j], q.means[3 * j + 1], q.means[3 * j + 2]));
    }
    T = t;
  }
  uint8_t *hist = &s_hist[warp][0][lane];
  for (int b = 0; b < kSelBins; ++b) hist[32 * b] = 0;
  const double invw = T > 0.0 ? (double)kSelBins / T : 0.0;
  auto bin_of = [&](double d2) {
    const double f = d2 * invw;
    return f >= (double)(kSelBins - 1) ? kSelBins - 1 : (int)f;
  };
  CellPos cp;
  cp.init(x, g);
  const double inv_h2 = 1.0 / (g.h * g.h);
  (void)glo;
  // warp ring scan (as k_knn_query) visiting every candidate with d2 <= Tb of
  // this lane; visit(d2, id) runs for the lane's qualifying candidates
  auto ring_scan = [&](double Tb, auto &&visit, auto &&tighten) {
    float Tc = cells2_bound(Tb, inv_h2);
    for (int r = 0;; ++r) {
      int lo[3], hi[3];
      bool full = true;
      for (int d = 0; d < 3; ++d) {
        lo[d] = blo[d] - r;
        hi[d] = bhi[d] + r;
        full = full && lo[d] <= 0 && hi[d] >= dims[d] - 1;
      }
      const int zlo = max(lo[2], 0), zhi = min(hi[2], dims[2] - 1);
      const int ylo = max(lo[1], 0), yhi = min(hi[1], dims[1] - 1);
      const int xlo = max(lo[0], 0), xhi = min(hi[0], dims[0] - 1);
      const int ny = yhi - ylo + 1, nslots = 2 * ny * (zhi - zlo + 1);
      for (int sb = 0; sb < nslots; sb += 32) {
        const int sl = sb + lane;
        int sa = 1, sbx = 0, sy = 0, sz = 0, se0 = 0, se1 = 0;
        if (sl < nslots) {
          const int ri = sl >> 1, side = sl & 1;
          sz = zlo + ri / ny;
          sy = ylo + ri - (ri / ny) * ny;
          const bool shell = r == 0 || sz == lo[2] || sz == hi[2] || sy == lo[1] || sy == hi[1];
          if (shell) {
            if (side == 0) sa = xlo, sbx = xhi;
          } else if (side == 0) {
            if (lo[0] >= 0) sa = sbx = lo[0];
          } else if (hi[0] <= dims[0] - 1) {
            sa = sbx = hi[0];
          }
          if (sa <= sbx) {
            const int64_t row = ((int64_t)sz * dims[1] + sy) * dims[0];
            se0 = g.cell_start[row + sa];
            se1 = g.cell_start[row + sbx + 1];
          }
        }
        const int cnt = min(32, nslots - sb);
        for (int jj = 0; jj < cnt; ++jj) {
          const int e0 = __shfl_sync(0xffffffffu, se0, jj), e1 = __shfl_sync(0xffffffffu, se1, jj);
          if (e0 >= e1) continue;
          const int a0 = __shfl_sync(0xffffffffu, sa, jj), b0 = __shfl_sync(0xffffffffu, sbx, jj);
          const int yy = __shfl_sync(0xffffffffu, sy, jj), zz = __shfl_sync(0xffffffffu, sz, jj);
          const bool need = Tb >= 0.0 && cp.box_d2(a0, b0, yy, zz, dims) <= Tc;
          if (!__any_sync(0xffffffffu, need)) continue;
          int e = e0;
          constexpr int KU = GSVR_SEL_UNROLL;  // 2: no spills at 72 registers (4 spilled: 12.1 vs 11.9 ms at cfg2)
          for (; e + KU <= e1; e += KU) {
            double4 c4[KU];
#pragma unroll
            for (int u = 0; u < KU; ++u) c4[u] = g.pts[e + u];
#pragma unroll
            for (int u = 0; u < KU; ++u) {
              const double d2 = dist2(c4[u].x, c4[u].y, c4[u].z);
              if (need && d2 <= Tb) visit(d2, (int)c4[u].w);
            }
          }
          for (; e < e1; ++e) {
            const double4 cand = g.pts[e];
            const double d2 = dist2(cand.x, cand.y, cand.z);
            if (need && d2 <= Tb) visit(d2, (int)cand.w);
          }
        }
      }
      const double tb = tighten(Tb);  // a lane's bound may shrink once its bins below it are complete
      if (tb < Tb) Tb = tb, Tc = cells2_bound(Tb, inv_h2);
      const double gap = (double)r * g.h * (1.0 - 1e-9);
      const bool done = Tb < 0.0 || full || Tb < gap * gap;
      if (__all_sync(0xffffffffu, done)) break;
    }
  };
  auto keep = [](double Tb) { return Tb; };
  // ---- pass 1: histogram of d2 <= T -------------------------------------
  // After each ring the lane's bound drops to the upper edge of the bin where
  // its cumulative count reaches kk: every later candidate below that edge is
  // still visited (rows are pruned against the current bound, the scan stops
  // only past it), so bins up to that edge stay complete, b* can only lie at or
  // below it, and bins above it are never read.
  bool sat = false;
  ring_scan(T, [&](double d2, int) {
    uint8_t &h = hist[32 * bin_of(d2)];
    sat |= h == 255;
    h += 1;
  }, [&](double Tb) {
    if (!(Tb > 0.0)) return Tb;
    int cum = 0;
    for (int b = 0; b < kSelBins; ++b) {
      cum += hist[32 * b];
      if (cum >= kk) return fmin(Tb, (double)(b + 1) * (T / kSelBins) * (1.0 + 1e-9));
    }
    return Tb;
  });
  int bstar = -1, clo = 0, nb = 0;
  if (active && sat) {  // a u8 counter wrapped: heap kernel
    fb_rows[atomicAdd(fb_count, 1)] = (int32_t)i;
    active = false;
  }
  if (active) {
    int cum = 0;
    for (int b = 0; b < kSelBins; ++b) {
      const int h = hist[32 * b];
      if (cum + h >= kk) {
        bstar = b;
        nb = h;
        break;
      }
      cum += h;
    }
    clo = cum;
    if (bstar < 0 || nb > kSelCap) {  // hand the row to the heap kernel
      fb_rows[atomicAdd(fb_count, 1)] = (int32_t)i;
      active = false;
    } else {
      int pos = 0;  // bins < b*: counters -> write cursors
      for (int b = 0; b < bstar; ++b) {
        const int h = hist[32 * b];
        hist[32 * b] = (uint8_t)pos;
        pos += h;
      }
    }
  }
  // ---- pass 2: place bins < b*, collect bin b* ---------------------------
  int32_t *orow = out + i * K;
  double *srow = scr + (i - row0) * kk;  // scratch rows of this launch
  double *bd = &s_bd[warp][0][lane];
  int32_t *bi = &s_bi[warp][0][lane];
  int nbl = 0;
  const double T2 = active ? fmin(T, (double)(bstar + 1) * (T / kSelBins) * (1.0 + 1e-9)) : -1.0;
  ring_scan(T2, [&](double d2, int id) {
    const int b = bin_of(d2);
    if (b < bstar) {
      const int p = hist[32 * b];
      hist[32 * b] = (uint8_t)(p + 1);
      orow[p] = id;  // p < clo <= K - 1 + (kk - K) ... always inside the K-row (clo < kk)
      srow[p] = d2;
    } else if (b == bstar) {
      bd[32 * nbl] = d2;
      bi[32 * nbl] = id;
      ++nbl;
    }
  }, keep);
  if (active) {
    GSVR_DCHECK(nbl == nb, "knn select boundary", nbl, nb);
    // boundary bin: sort by (d2, id); its first kk - clo entries complete the row
    for (int u = 1; u < nbl; ++u) {
      const double dv = bd[32 * u];
      const int iv = bi[32 * u];
      int v = u;
      while (v > 0 && knn_less(dv, iv, bd[32 * (v - 1)], bi[32 * (v - 1)])) {
        bd[32 * v] = bd[32 * (v - 1)];
        bi[32 * v] = bi[32 * (v - 1)];
        --v;
      }
      bd[32 * v] = dv;
      bi[32 * v] = iv;
    }
    for (int u = 0; clo + u < kk; ++u) {
      const int p = clo + u;
      if (p < K) orow[p] = bi[32 * u];
      else q.out_next[i] = bi[32 * u];
      srow[p] = bd[32 * u];
    }
  }
  __syncwarp();  // rows complete in global memory -> visible to the whole warp
  // ---- per row, warp-cooperative: finish the (d2, id) order inside bins and
  // apply the knn.py:58-74 rules.  Lane l holds positions 2l, 2l+1; the row is
  // bin-sorted, so an odd-even transposition sort ends after ~max-bin rounds.
  auto same_dist = [](double lo_, double hi_) {
    if (hi_ == lo_) return true;
    if (hi_ > lo_ * (1.0 + 1e-14)) return false;
    return sqrt(lo_) == sqrt(hi_);
  };
  const int64_t wbase = i - lane;
  const int p0 = 2 * lane, p1 = 2 * lane + 1;
  const unsigned act = __ballot_sync(0xffffffffu, active);
  // the next active row's entries are loaded while this row is being ordered
  auto load_row = [&](int r, double &d0, int &i0, double &d1, int &i1) {
    const int64_t ir = wbase + r;
    const int32_t *orr = out + ir * K;
    const double *srr = scr + (ir - row0) * kk;
    d0 = d1 = INFINITY;
    i0 = i1 = INT32_MAX;
    if (p0 < kk) d0 = srr[p0], i0 = p0 < K ? orr[p0] : q.out_next[ir];
    if (p1 < kk) d1 = srr[p1], i1 = p1 < K ? orr[p1] : q.out_next[ir];
  };
  double nd0 = INFINITY, nd1 = INFINITY;
  int ni0 = INT32_MAX, ni1 = INT32_MAX;
  if (act) load_row(__ffs(act) - 1, nd0, ni0, nd1, ni1);
  for (unsigned rows = act; rows;) {
    const int r = __ffs(rows) - 1;
    rows &= rows - 1;
    const int64_t ir = wbase + r;
    int32_t *orr = out + ir * K;
    double *srr = scr + (ir - row0) * kk;
    int32_t *nxt = q.out_next + ir;
    double d0 = nd0, d1 = nd1;
    int i0 = ni0, i1 = ni1;
    if (rows) load_row(__ffs(rows) - 1, nd0, ni0, nd1, ni1);
    for (;;) {
      bool sw = false;
      if (knn_less(d1, i1, d0, i0)) {  // even phase: (2l, 2l+1)
        const double td = d0; d0 = d1; d1 = td;
        const int ti = i0; i0 = i1; i1 = ti;
        sw = true;
      }
      // odd phase: (2l+1, 2l+2) across lanes l, l+1
      const double dn = __shfl_down_sync(0xffffffffu, d0, 1), dp = __shfl_up_sync(0xffffffffu, d1, 1);
      const int in = __shfl_down_sync(0xffffffffu, i0, 1), ip = __shfl_up_sync(0xffffffffu, i1, 1);
      const bool hi_sw = lane < 31 && knn_less(dn, in, d1, i1);
      const bool lo_sw = lane > 0 && knn_less(d0, i0, dp, ip);
      if (hi_sw) d1 = dn, i1 = in, sw = true;
      if (lo_sw) d0 = dp, i0 = ip;
      if (!__any_sync(0xffffffffu, sw)) break;
    }
    auto at_d = [&](int p) { return __shfl_sync(0xffffffffu, (p & 1) ? d1 : d0, p >> 1); };
    const bool tie = kk > K && same_dist(at_d(K - 1), at_d(K));
    bool runs = false;
    if (!tie) {  // any equal-sqrt neighbours -> the id reordering of knn.py:58-74
      const double dprev = __shfl_up_sync(0xffffffffu, d1, 1);
      const bool f0 = p0 >= 1 && p0 < kk && same_dist(dprev, d0);
      const bool f1 = p1 < kk && same_dist(d0, d1);
      runs = __any_sync(0xffffffffu, f0 || f1);
    }
    if (p0 < kk) (p0 < K ? orr[p0] : *nxt) = i0, srr[p0] = d0;
    if (p1 < kk) (p1 < K ? orr[p1] : *nxt) = i1, srr[p1] = d1;
    if (runs) {  // rare (exact or sqrt-level distance ties): the heap kernel's sequential rule
      __syncwarp();
      if (lane == 0) {
        auto ID = [&](int p) -> int32_t & { return p < K ? orr[p] : *nxt; };
        int a = 0;
        while (a < K) {
          int b = a + 1;
          while (b < kk && same_dist(srr[b - 1], srr[b])) ++b;
          for (int u = a + 1; u < b; ++u) {
            const int id = ID(u);
            const double dv = srr[u];
            int v = u;
            while (v > a && ID(v - 1) > id) {
              ID(v) = ID(v - 1);
              srr[v] = srr[v - 1];
              --v;
            }
            ID(v) = id;
            srr[v] = dv;
          }
          a = b;
        }
      }
      __syncwarp();
    }
    if (kk <= K && lane == 0) *nxt = -1;
  }
}

// GSVR_KNN_SEEDS=0 disables refresh seeding (A/B timing; results are identical)
static bool getenv_seeds_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_KNN_SEEDS");
    return !(v && v[0] == '0');
  }();
  return on;
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
  // one warp per block: the per-thread heaps (12 B per kept candidate) fill
  // shared memory, and 32-thread blocks pack it tightest (11 warps per SM)
  const size_t sm = per * 32;
  if (sm <= limit) {
    GSVR_TRY(ensure_smem((const void *)k_knn_query<32>, sm));
#ifdef GSVR_KNN_STATS
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    cudaMemcpyToSymbolAsync(g_knn_stats, z, sizeof(z), 0, cudaMemcpyHostToDevice, st);
#endif
    const unsigned nblk = q.one_per_warp ? (unsigned)q.M : (unsigned)((q.M + 31) / 32);
    k_knn_query<32><<<nblk, 32, sm, st>>>(q, g, (int)K, kk, out, out_i64);
    GSVR_LAUNCH_CHECK("k_knn_query");
#ifdef GSVR_KNN_STATS
    cudaMemcpyFromSymbolAsync(z, g_knn_stats, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
    cudaStreamSynchronize(st);
    fprintf(stderr, "KNNSTATS M=%lld warps=%llu cand/warp=%.1f rows/warp=%.1f skipped/warp=%.1f siftup/q=%.1f "
            "siftdown/q=%.1f rings/warp=%.2f under/q=%.1f seeded=%d h=%g dims=%dx%dx%d\n",
            (long long)q.M, z[0], (double)z[1] / z[0], (double)z[2] / z[0], (double)z[3] / z[0],
            (double)z[4] / q.M, (double)z[5] / q.M, (double)z[6] / z[0], (double)z[7] / q.M, q.seed != nullptr,
            g.h, g.d0, g.d1, g.d2);
#endif
    return GSVR_OK;
  }
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
  static const double per_cell = [] {
    const char *v = std::getenv("GSVR_KNN_PER_CELL");
    return v ? std::max(0.1, std::atof(v)) : 3.0;
  }();
  double h = emax > 0 ? std::pow(vol * per_cell / (double)N, 1.0 / std::max(nd, 1)) : 1.0;
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
  if (cudaMallocAsync((void **)&ix->means, N * 24, st) != cudaSuccess)
    return bail(fail(GSVR_ERR_CUDA, "out of device memory for the K-NN index"));
  cudaMemcpyAsync(ix->means, means, N * 24, cudaMemcpyDeviceToDevice, st);
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
  QuerySrc q{sorted.as<double>(), nullptr, nullptr, nullptr, nullptr, order.as<int32_t>(), M,
             nullptr, nullptr, nullptr, nullptr};
  return knn_run(ix, q, K, out, out_i64, st);
}

__global__ void k_spatial_pos(int64_t N, const double4 *__restrict__ pts, int32_t *__restrict__ gpos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    gpos[(int64_t)pts[i].w] = (int32_t)i;
}

// GSVR_GPOS=0 keeps the tile kernel's packed rows in id order (A/B; results identical)
static bool gpos_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_GPOS");
    return !(v && v[0] == '0');
  }();
  return on;
}

// GSVR_KNN_SELECT=0 runs the heap kernel for seeded refreshes too (A/B timing; results identical)
static bool select_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_KNN_SELECT");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Seeded batch refresh through k_knn_select; rows it hands back (boundary bin
// over capacity) go through the heap kernel with their seeds.
static int knn_select_run(gsvr_batch *b, const gsvr_knn_index *ix, const QuerySrc &q, int64_t K, cudaStream_t st) {
  const int kk = (int)std::min<int64_t>(K + 1, ix->N);
  GridView g{ix->lo[0], ix->lo[1], ix->lo[2], ix->h, ix->dims[0], ix->dims[1], ix->dims[2], ix->pts,
             ix->cell_start};
  // rows in launches of <= 2^21 (d2 scratch of one launch: ~0.9 GB at K = 50, reused)
  const int64_t chunk = std::min<int64_t>(b->P, 1 << 21);
  GSVR_TRY(grow(b->ws_knn_scr, b->ws_knn_scr_cap, (size_t)chunk * kk * 8, st));
  GSVR_TRY(grow(b->ws_knn_fb, b->ws_knn_fb_cap, (size_t)b->P * 4 + 16, st));
  int *fb_count = reinterpret_cast<int *>(b->ws_knn_fb);
  int32_t *fb_rows = reinterpret_cast<int32_t *>(b->ws_knn_fb) + 4;
  GSVR_CUDA(cudaMemsetAsync(fb_count, 0, 4, st));
  for (int64_t r0 = 0; r0 < q.M; r0 += chunk) {
    QuerySrc qc = q;
    qc.M = std::min<int64_t>(q.M, r0 + chunk);
    const unsigned blocks = (unsigned)((qc.M - r0 + 32 * kSelWarps - 1) / (32 * kSelWarps));
    k_knn_select<kSelWarps><<<blocks, 32 * kSelWarps, 0, st>>>(qc, g, (int)K, kk, b->nbr_int,
                                                               reinterpret_cast<double *>(b->ws_knn_scr), r0,
                                                               fb_rows, fb_count);
    GSVR_LAUNCH_CHECK("k_knn_select");
  }
  int nfb = 0;
  GSVR_CUDA(cudaMemcpyAsync(&nfb, fb_count, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  b->knn_fallback_rows = nfb;
  if (trace_enabled()) std::fprintf(stderr, "[gsvr trace] knn/select fallback rows %d of %lld\n", nfb, (long long)q.M);
  if (nfb > 0) {
    QuerySrc qf = q;
    qf.rows = fb_rows;
    qf.M = nfb;
    qf.one_per_warp = 1;  // fallback rows are scattered: each gets its own warp box
    GSVR_TRY(knn_run(ix, qf, K, b->nbr_int, 0, st));
  }
  return GSVR_OK;
}

int64_t gsvr_batch_knn_fallback_rows(const gsvr_batch *b) { return b ? b->knn_fallback_rows : -1; }

void gsvr_batch_invalidate_seeds(gsvr_batch *b) {
  if (b) b->seeds_valid = false;
}

int gsvr_batch_refresh(gsvr_batch *b, const gsvr_knn_index *ix, int64_t K, const double *Rc, const double *tvec,
                       void *stream) {
  cudaStream_t st = as_stream(stream);
  b->knn_fallback_rows = -1;  // -1: the last refresh did not run the selection kernel
  if (b->nbr_int && b->K != K) b->release_binning();
  if (!b->nbr_int) GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_int, b->P * K * 4, st));
  if (!b->nbr_next) GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_next, b->P * 4, st));
  StageTrace tr("refresh", st);
  // seeds: the previous refresh's lists (same K, same N, our own distinct ids);
  // each row reads its seeds before its own thread overwrites them
  const bool seeded = b->seeds_valid && b->K == K && b->seeds_N == ix->N && getenv_seeds_enabled();
  QuerySrc q{nullptr, b->x0s, b->sid_s, Rc, tvec, nullptr, b->P,
             seeded ? b->nbr_int : nullptr, seeded ? b->nbr_next : nullptr, ix->means, b->nbr_next};
  b->seeds_valid = false;
  if (seeded && select_enabled())
    GSVR_TRY(knn_select_run(b, ix, q, K, st));
  else
    GSVR_TRY(knn_run(ix, q, K, b->nbr_int, 0, st));
  tr.mark("knn");
  // packed-row positions for the tile kernel in the index's cell order
  if (gpos_enabled()) {
    GSVR_TRY(grow(b->gpos, b->cap_gpos, (size_t)ix->N * 4 + 16, st));
    k_spatial_pos<<<grid_for(ix->N, 256), 256, 0, st>>>(ix->N, ix->pts, b->gpos);
    GSVR_LAUNCH_CHECK("k_spatial_pos");
    b->gpos_N = ix->N;
  } else {
    b->gpos_N = 0;
  }
  GSVR_TRY(batch_bin_internal(b, K, ix->N, st));
  tr.mark("bin");
  b->seeds_valid = true;
  b->seeds_N = ix->N;
  return GSVR_OK;
}

}  // extern "C"
