// batch.cuh -- the device-resident point batch and its (slice, tile) binning.
//
// HBM layout (all "internal order" = points sorted by (slice, Morton code of
// the nominal position), cut into single-slice tiles of <= tile_points):
//   perm[P]          int32   internal -> caller index
//   sid_s[P]         int32   slice id, internal order
//   x0s[P]           double3 nominal positions (fp64, for K-NN refresh / staleness)
//   d0obs[P]         float4  (x0 - tile_origin, I_obs) -- tile-relative fp32 offsets
//   iobs_s[P]        double  I_obs (float64; read only for ambiguous L1 signs)
//   tile_start[T]    int64, tile_n[T] int32, tile_slice[T] int32, tile_origin[T] double3
// Binning (refreshed with the neighbour lists; K fixed per binning):
//   nbr_int[P*K]     int32   global ids, internal order, row-major (the K-NN output)
//   nbr_local[P*K]   uint16  per tile, k-major: local id of pair (p, k)
//   pair_pix[P*K]    uint16  per tile, Gaussian-major pair list: pixel of each pair
//   uoff[T+1]        int32   offsets of each tile's unique-Gaussian list
//   gid[U]           int32   unique global ids per tile (ascending)
//   csr[U+T]         uint16  per tile: first pair of each local Gaussian (+ sentinel)
#pragma once

#include <vector>

#include "common.cuh"

struct gsvr_batch {
  int64_t P = 0, S = 0, T = 0;
  int TP = 0;
  int32_t *perm = nullptr;
  int32_t *sid_s = nullptr;
  double *x0s = nullptr;
  float4 *d0obs = nullptr;
  double *iobs_s = nullptr;  // (P) observed intensities in float64 (sign refinement of ambiguous residuals)
  int64_t *tile_start = nullptr;
  int32_t *tile_n = nullptr;
  int32_t *tile_slice = nullptr;
  double *tile_origin = nullptr;
  double *tile_radius = nullptr;  // (T) max |x0 - origin| over the tile (staleness bounds)
  // slice-plane geometry: every tile of a real slice is planar; then each point
  // is o_t + alpha b1_t + beta b2_t exactly (to 1e-8 mm) and the planar kernel runs
  double *tile_basis = nullptr;  // (T, 6): b1, b2 orthonormal in-plane axes (nominal frame)
  float2 *ab = nullptr;          // (P): in-plane coordinates (alpha, beta), fp32
  bool planar = false;
  // binning
  int64_t K = 0, N = 0, U = 0;
  int max_unique = 0;
  int32_t *nbr_int = nullptr;
  // K-NN refresh seeds: the (K+1)-th neighbour of the last device refresh; with
  // the K lists it is a set of kk distinct means whose distances under the new
  // positions bound every point's kk-th distance (exact pruning, knn.cu)
  int32_t *nbr_next = nullptr;  // (P)
  bool seeds_valid = false;     // nbr_int/nbr_next came from gsvr_batch_refresh with (K, N)
  int64_t seeds_N = 0;
  uint16_t *nbr_local = nullptr;  // per tile at nl_off[t] (16-byte aligned, TMA bulk source)
  uint16_t *pair_pix = nullptr;   // per tile at pp_off[t], chunk-transposed: pair c*C+r at r*256+c
  int64_t *nl_off = nullptr;      // (T+1)
  int64_t *pp_off = nullptr;      // (T+1)
  std::vector<int64_t> h_tstart;  // host copies of the tile table
  std::vector<int32_t> h_tn;
  int32_t *uoff = nullptr;
  int32_t *gid = nullptr;
  uint16_t *csr = nullptr;
  float4 *rec = nullptr;  // per (tile, unique Gaussian) records; only used by tiles exceeding one page
  // deterministic per-Gaussian gradient reduction: every (tile, Gaussian) record
  // writes its 10 partial sums to gpart[u]; jr_ptr/jr_idx list, per Gaussian j,
  // its records u in tile order, and k_gather_grads sums them in that order.
  float *gpart = nullptr;   // (U, 10)
  double *tpart = nullptr;  // (T, 20) per-tile slice-gradient partials (summed per slice in tile order)
  int32_t *slice_tile0 = nullptr;  // (S + 1) first tile of each slice
  int32_t *jr_ptr = nullptr;  // (N + 1)
  int32_t *jr_idx = nullptr;  // (U)
  int32_t *gorder = nullptr;  // (N) Gaussians by their first record (memory locality of the gather)
  // spatial position of every Gaussian's packed row for the tile kernel: the
  // K-NN index's cell order at the last device refresh (a tile's Gaussians
  // then sit in a few contiguous runs of rows); valid while gpos_N == N
  int32_t *gpos = nullptr;
  int64_t gpos_N = 0;
  size_t cap_gpos = 0;
  uint8_t *rot_flag = nullptr;  // (T) tiles binned by a sorting path: pair order rotated in bin_finish
  size_t cap_rot_flag = 0;
  // Binning buffers only grow (with headroom), and the per-tile layout
  // (nl_off/pp_off/nbr_local/pair_pix) depends only on the tiles and K, so a
  // steady-state refresh never goes back to the allocator.
  int64_t layout_K = 0;
  size_t cap_gid = 0, cap_csr = 0, cap_rec = 0, cap_gpart = 0, cap_jr_idx = 0, cap_jr_ptr = 0, cap_gorder = 0;
  void *ws[6] = {nullptr, nullptr, nullptr, nullptr, nullptr, nullptr};  // binning workspace
  mutable void *ws_disp = nullptr;  // staleness bounds (T doubles + lower bound)
  mutable void *ws_grec = nullptr;  // packed (mu, c, cov6) per Gaussian for the tile kernel
  void *ws_knn_scr = nullptr;       // seeded K-NN selection: (P, kk) d2 scratch
  size_t ws_knn_scr_cap = 0;
  void *ws_knn_fb = nullptr;        // seeded K-NN selection: fallback row list (+ count)
  size_t ws_knn_fb_cap = 0;
  int64_t knn_fallback_rows = 0;    // rows of the last seeded refresh handed to the heap kernel
  mutable size_t ws_grec_cap = 0;
  mutable size_t ws_disp_cap = 0;
  mutable void *ws_brec = nullptr;  // (U, 3) float4 backward record halves of large-tile launches
  mutable size_t ws_brec_cap = 0;
  size_t ws_cap[6] = {0, 0, 0, 0, 0, 0};
  cudaStream_t owner_stream = nullptr;
  // per-tile unique counts of the last binning (host) and the tile kernel's
  // launch buckets built from them: tiles whose records fit a page that keeps
  // full residency, and the rest (train_planar.cu)
  std::vector<int32_t> h_nu;
  mutable bool buckets_valid = false;
  mutable int bucket_cap = 0;
  mutable int32_t *tile_buckets = nullptr;  // [small tiles | large tiles]
  mutable int64_t n_small = 0, n_large = 0;
  mutable size_t cap_tile_buckets = 0;
  void release_binning();
  ~gsvr_batch();
};

namespace gsvr {
constexpr int kChunkThreads = 256;
// the smallest shared-memory record page of the tile kernels (planar kPCap,
// general kRecCap): tiles with at most this many unique Gaussians never read
// the global record pages
constexpr int kMinRecordPage = 1536;  // backward chunks per tile (= threads of the tile kernels)
// Gaussian-major pair list layout: chunk c (= thread) owns pairs [c*C, (c+1)*C);
// its r-th pair sits at ((r/8)*256 + c)*8 + r%8, so a thread fetches 8 pairs with
// one 16-byte load and a warp's loads are contiguous.
__host__ __device__ inline int chunk_len(int m) { return (m + kChunkThreads - 1) / kChunkThreads; }
__host__ __device__ inline int chunk_stride(int m) { return (chunk_len(m) + 7) / 8 * 8; }
__host__ __device__ inline int64_t pair_slot(int i, int C) {
  const int c = i / C, r = i - c * C;
  return ((int64_t)(r >> 3) * kChunkThreads + c) * 8 + (r & 7);
}
// i / d for 0 <= i, i * d < 2^32 via one wide multiply: M = ceil(2^32 / d)
__host__ __device__ inline uint64_t div_magic(int d) { return ((1ull << 32) + (uint64_t)d - 1) / (uint64_t)d; }
__host__ __device__ inline int div_by(int i, uint64_t M) { return (int)(((uint64_t)(uint32_t)i * M) >> 32); }
// nbr_local layout per tile (n pixels, K neighbours): k-PAIR-major, element
// (p, k) at ((k/2)*n + p)*2 + k%2, so a pixel reads the local ids of neighbours
// k and k+1 with one 32-bit load; K odd leaves one padding slot per pixel.
__host__ __device__ inline int64_t nl_index(int p, int k, int n) {
  return ((int64_t)(k >> 1) * n + p) * 2 + (k & 1);
}
__host__ __device__ inline int64_t nl_len(int n, int K) { return (int64_t)((K + 1) >> 1) * 2 * n; }
// Grow-only device buffer: reallocates (25% headroom) only when need > cap.
template <class T>
inline int grow(T *&p, size_t &cap, size_t need, cudaStream_t st) {
  if (p && cap >= need) return GSVR_OK;
  if (p) cudaFreeAsync(p, st), p = nullptr;
  const size_t nb = need + need / 4 + 256;
  GSVR_CUDA(cudaMallocAsync((void **)&p, nb, st));
  cap = nb;
  return GSVR_OK;
}
// Shared by the drop-in train call and the fit loop.
int batch_create(int64_t P, int64_t S, const double *x0, const int32_t *sid, const double *I_obs,
                 int tile_points, gsvr_batch **out, cudaStream_t st);
int batch_bin_internal(gsvr_batch *b, int64_t K, int64_t N, cudaStream_t st);
// binning in stages (the host-buffer drop-in pipelines it with the neighbour upload)
struct BinPlan {
  int bits = 0, pbits = 0;
  bool fast = false;  // per-tile shared-memory sort applies
  // deferred overflow (hash path): tiles the hash kernel hands to the sort are
  // collected here across several bin_sort_tiles calls, then bin_flush_overflow
  int32_t *ov_list = nullptr;
  int *ov_count = nullptr;
};
int bin_prepare(gsvr_batch *b, int64_t K, int64_t N, cudaStream_t st, BinPlan *plan);
// optional direct source of the neighbour ids: caller-order (P, K) rows read
// through perm (no nbr_int copy); out-of-range ids set *bad
struct BinSource {
  const void *nbr = nullptr;
  int i64 = 0;
  const int32_t *perm = nullptr;
  int64_t N = 0;
  int *bad = nullptr;
};
// tiles tile_list[t0..t1) (or t0..t1 when tile_list is null)
int bin_sort_tiles(gsvr_batch *b, int64_t K, const BinPlan &plan, int64_t t0, int64_t t1, cudaStream_t st,
                   const int32_t *tile_list = nullptr, BinSource ext = BinSource());
int bin_finish(gsvr_batch *b, int64_t K, int64_t N, const BinPlan &plan, cudaStream_t st);
int bin_flush_overflow(gsvr_batch *b, int64_t K, const BinPlan &plan, cudaStream_t st, BinSource ext);
// caller-order neighbour rows -> nbr_int (internal order) for internal rows [i0, i1);
// out-of-range ids set *bad (device flag)
int gather_nbr_rows(gsvr_batch *b, int64_t K, int64_t N, const void *nbr, int nbr_i64, int64_t i0, int64_t i1,
                    int *bad, cudaStream_t st);
int train_tiles(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                const double *cov6, const double *cvals, double delta, float *dfield,
                double *dslice, double *I_hat, double *absres, unsigned long long *nonfinite_first,
                cudaStream_t st);
int gather_grads(const gsvr_batch *b, float *dfield, double *dslice, cudaStream_t st);
int train_tiles_planar(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                       const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                       const double *cov6, const double *cvals, double delta, float *dfield, double *dslice,
                       double *I_hat, double *absres, unsigned long long *nonfinite_first, cudaStream_t st);
// ---- L1 sign refinement (kernels.py:133-143) ------------------------------
// The tile kernels render in fp32.  Where |r| = |I_hat - I_obs| is within the
// fp32 render tolerance (kResidualFloorRel of max(|I|, |I_hat|)) its sign is not
// resolved in fp32, so the pixel is re-rendered in float64 with the
// reference's per-pair formulation (world point Rc x0 + t, Sigma_j + Sigma_PSF,
// 3x3 inverse, drop below -80; kernels.py:103-132), one warp per ambiguous
// pixel (lanes split the K pairs).  The subgradient then follows the float64
// residual; only |r64| <= kResidualZeroRel * max(|I|, |I_hat|) -- far below
// any data precision, where the reference's own sign is its rounding noise --
// counts as the exact zero, which keeps an exact fit a fixed point.
constexpr float kResidualFloorRel = 1e-5f;
constexpr double kResidualZeroRel = 1e-12;

// Warp-cooperative float64 (num, den - delta) of pixel pp (internal index ip).
// nl: the tile's pixel-major local ids (nl_index layout), gid_t: the tile's
// unique global ids.  Every lane of the warp must call it with the same pp.
__device__ inline double2 refine_pixel_f64(int lane, int pp, int n, int K, const uint16_t *nl,
                                           const int32_t *gid_t, const double *x0s, int64_t ip,
                                           const double *R, const double *tv, const double *p6,
                                           const double *mu, const double *cov6, const double *cvals) {
  const double a0 = x0s[3 * ip], a1 = x0s[3 * ip + 1], a2 = x0s[3 * ip + 2];
  double x[3];
#pragma unroll
  for (int r = 0; r < 3; ++r)
    x[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[3 * r], a0), __dmul_rn(R[3 * r + 1], a1)),
                               __dmul_rn(R[3 * r + 2], a2)), tv[r]);
  double num = 0.0, den = 0.0;
  for (int k = lane; k < K; k += 32) {
    const int64_t j = gid_t[nl[nl_index(pp, k, n)]];
    double S6[6], M[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) S6[e] = cov6[6 * j + e] + p6[e];
    inv_sym3<double>(S6, M);
    const double v0 = x[0] - mu[3 * j], v1 = x[1] - mu[3 * j + 1], v2 = x[2] - mu[3 * j + 2];
    const double w0 = M[0] * v0 + M[1] * v1 + M[2] * v2;
    const double w1 = M[1] * v0 + M[3] * v1 + M[4] * v2;
    const double w2 = M[2] * v0 + M[4] * v1 + M[5] * v2;
    const double u = -0.5 * (v0 * w0 + v1 * w1 + v2 * w2);
    const double e = u < kExpClamp ? 0.0 : exp(u);
    num += cvals[j] * e;
    den += e;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    num += __shfl_xor_sync(0xffffffffu, num, o);
    den += __shfl_xor_sync(0xffffffffu, den, o);
  }
  return make_double2(num, den);
}

// Per-pixel L1 bookkeeping shared by the tile kernels: given the fp32 render
// (ratio = num/den) of pixel p (< n, else inactive), refines ambiguous signs in
// float64 (warp-collective: all 32 lanes call it) and returns the subgradient
// g (+-w or 0); ratio / ihat / r are replaced by their float64 values there.
struct PixelL1 {
  float ratio, ihat, r, g;
  double ihat_d, absr_d;  // outputs (float64 where refined)
};
__device__ inline PixelL1 pixel_l1(bool active, float num, float den, float iobs, float sig, float wdat, int pp,
                                   int n, int K, const uint16_t *nl, const int32_t *gid_t, const double *x0s,
                                   int64_t ts, const double *R, const double *tv, const double *p6,
                                   const double *mu, const double *cov6, const double *cvals, double sig64,
                                   double delta64, const double *iobs64) {
  PixelL1 o{0.f, 0.f, 0.f, 0.f, 0.0, 0.0};
  bool amb = false;
  if (active) {
    o.ratio = num / den;
    o.ihat = sig * o.ratio;
    o.r = o.ihat - iobs;
    amb = fabsf(o.r) <= kResidualFloorRel * fmaxf(fabsf(iobs), fabsf(o.ihat));
    o.g = (o.r > 0.f) ? wdat : -wdat;
    o.ihat_d = (double)o.ihat;
    o.absr_d = (double)fabsf(o.r);
  }
  const int lane = threadIdx.x & 31;
#ifdef GSVR_NO_REFINE  // diagnostics only: fp32 sign everywhere (timing A/B of the refinement)
  unsigned ball = 0;
  (void)amb;
#else
  unsigned ball = __ballot_sync(0xffffffffu, amb);
#endif
  while (ball) {
    const int src = __ffs(ball) - 1;
    ball &= ball - 1;
    const int q = (pp & ~31) + src;
    const double2 nd = refine_pixel_f64(lane, q, n, K, nl, gid_t, x0s, ts + q, R, tv, p6, mu, cov6, cvals);
    if (lane == src) {
      const double ratio64 = nd.x / (nd.y + delta64);
      const double ihat64 = sig64 * ratio64;
      const double io = iobs64[ts + q];
      const double r64 = ihat64 - io;
      o.ratio = (float)ratio64;
      o.ihat = (float)ihat64;
      o.r = (float)r64;
      o.ihat_d = ihat64;
      o.absr_d = fabs(r64);
      o.g = fabs(r64) <= kResidualZeroRel * fmax(fabs(io), fabs(ihat64)) ? 0.f : (r64 > 0.0 ? wdat : -wdat);
    }
  }
  return o;
}

// sortable uint64 keys for doubles (min/max reductions with integer atomics)
__host__ __device__ inline unsigned long long dkey(double x) {
#ifdef __CUDA_ARCH__
  unsigned long long u = (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long u;
  memcpy(&u, &x, 8);
#endif
  return (u >> 63) ? ~u : (u | 0x8000000000000000ull);
}
__host__ __device__ inline double dkey_inv(unsigned long long k) {
  unsigned long long u = (k >> 63) ? (k & 0x7fffffffffffffffull) : ~k;
#ifdef __CUDA_ARCH__
  return __longlong_as_double((long long)u);
#else
  double x;
  memcpy(&x, &u, 8);
  return x;
#endif
}
// Bounding box of n points (stride 3 doubles): keys[0..2] = min, keys[3..5] = max.
int bbox3(const double *pts, int64_t n, unsigned long long *keys_dev, double out_host[6],
          cudaStream_t st);
// Spread the low 21 bits of v over every third bit.
__host__ __device__ inline unsigned long long spread3(unsigned long long v) {
  v &= 0x1fffffull;
  v = (v | v << 32) & 0x1f00000000ffffull;
  v = (v | v << 16) & 0x1f0000ff0000ffull;
  v = (v | v << 8) & 0x100f00f00f00f00full;
  v = (v | v << 4) & 0x10c30c30c30c30c3ull;
  v = (v | v << 2) & 0x1249249249249249ull;
  return v;
}
}  // namespace gsvr
