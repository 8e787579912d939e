// init.cu -- the fit's setup on the device.
//
//  * the point batch (motion.py:183-237 build_point_batch): every masked pixel
//    in stack -> slice -> raster (u, v) order, lifted to world mm, with its
//    slice id and value;
//  * the content-adaptive initial cloud (initialization.py:44-152): in-plane
//    gradient magnitudes, numpy's Generator.choice(P, N, p=prob) over the
//    pooled masked pixels (weights -> pairwise total -> probabilities ->
//    cumulative distribution -> searchsorted of the host's PCG64 uniforms), the
//    lifting of the drawn pixels and each position's source-stack intensity.
//
// Bit-identical to the reference's numpy on the same host, by construction:
//  * np.gradient: (f[i+1] - f[i-1]) / 2 inside, one-sided differences at the
//    edges; np.hypot is glibc 2.39's hypot (e_hypot.c, non-FMA build: Borges'
//    corrected sqrt), restated below with explicitly rounded operations -- not
//    CUDA's hypot, which rounds differently in ~0.5 % of cases;
//  * ndarray.sum: numpy's pairwise summation (blocks of <= 128 summed with 8
//    accumulators, halves rounded down to multiples of 8), evaluated as a
//    bottom-up tree on the device;
//  * cumsum: add.accumulate is a sequential chain of rounded adds, and the
//    chain's rounding is what the draw boundaries are made of, so one thread
//    runs it, fed and drained by TMA bulk copies through a shared-memory ring;
//  * x @ A[:3, :3].T + A[:3, 3] is OpenBLAS dgemm on (m, 3) x (3, 3): per
//    element fma(x2, a2, fma(x1, a1, x0 * a0)) -- for m == 1 numpy calls gemv,
//    whose order is fma(x2, a2, fma(x0, a0, x1 * a1)) -- then the translation.
//    (OpenBLAS 0.3.30 SkylakeX kernels as shipped with numpy 2.3 in this image;
//    tests/test_gpu_init.py pins every output against numpy on the GPU host.)
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <cmath>
#include <vector>

#include "common.cuh"
#include "tma.cuh"

namespace gsvr {

constexpr int kMaxStacks = 64;

struct StackTab {
  int n;
  int64_t nx[kMaxStacks], ny[kMaxStacks], ns[kMaxStacks];
  const double *data[kMaxStacks];
  const uint8_t *mask[kMaxStacks];
  double A[kMaxStacks][12];  // affine rows 0..2
  int64_t slice0[kMaxStacks + 1];  // first global slice of each stack
  int64_t pool0[kMaxStacks + 1];   // first pooled (C-order masked) index of each stack
};

__device__ __forceinline__ int stack_of_slice(const StackTab &t, int64_t s) {
  int k = 0;
  while (k + 1 < t.n && t.slice0[k + 1] <= s) ++k;
  return k;
}

// x @ A[:3, :3].T + A[:3, 3] for one row x of an (m, 3) product (header comment)
__device__ __forceinline__ void affine_row(const double *A, double x0, double x1, double x2, bool gemv,
                                           double out[3]) {
#pragma unroll
  for (int j = 0; j < 3; ++j) {
    const double *a = A + 4 * j;
    const double s = gemv ? __fma_rn(x2, a[2], __fma_rn(x0, a[0], __dmul_rn(x1, a[1])))
                          : __fma_rn(x2, a[2], __fma_rn(x1, a[1], __dmul_rn(x0, a[0])));
    out[j] = __dadd_rn(s, a[3]);
  }
}

// glibc 2.39 sysdeps/ieee754/dbl-64/e_hypot.c, the non-FMA kernel (what numpy's
// np.hypot calls on x86-64), every operation explicitly rounded
__device__ double glibc_hypot_kernel(double ax, double ay) {
  double h = __dsqrt_rn(__dadd_rn(__dmul_rn(ax, ax), __dmul_rn(ay, ay)));
  double t1, t2;
  if (h <= __dmul_rn(2.0, ay)) {
    const double delta = __dsub_rn(h, ay);
    t1 = __dmul_rn(ax, __dsub_rn(__dmul_rn(2.0, delta), ax));
    t2 = __dmul_rn(__dsub_rn(delta, __dmul_rn(2.0, __dsub_rn(ax, ay))), delta);
  } else {
    const double delta = __dsub_rn(h, ax);
    t1 = __dmul_rn(__dmul_rn(2.0, delta), __dsub_rn(ax, __dmul_rn(2.0, ay)));
    t2 = __dadd_rn(__dmul_rn(__dsub_rn(__dmul_rn(4.0, delta), ay), ay), __dmul_rn(delta, delta));
  }
  return __dsub_rn(h, __ddiv_rn(__dadd_rn(t1, t2), __dmul_rn(2.0, h)));
}

__device__ double glibc_hypot(double x, double y) {
  const double kScale = 0x1p-600, kLarge = 0x1p+511, kTiny = 0x1p-511, kEps = 0x1p-54;
  if (!isfinite(x) || !isfinite(y)) {
    if (isinf(x) || isinf(y)) return INFINITY;
    return __dadd_rn(x, y);
  }
  x = fabs(x);
  y = fabs(y);
  double ax = x < y ? y : x, ay = x < y ? x : y;
  if (ax > kLarge) {
    if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
    return __ddiv_rn(glibc_hypot_kernel(__dmul_rn(ax, kScale), __dmul_rn(ay, kScale)), kScale);
  }
  if (ay < kTiny) {
    if (ax >= __ddiv_rn(ay, kEps)) return __dadd_rn(ax, ay);
    return __dmul_rn(glibc_hypot_kernel(__ddiv_rn(ax, kScale), __ddiv_rn(ay, kScale)), kScale);
  }
  if (ay <= __dmul_rn(ax, kEps)) return __dadd_rn(ax, ay);
  return glibc_hypot_kernel(ax, ay);
}

// ---- masked pixels per slice, and the point batch ----------------------------
// One block per (stack, slice): the slice's raster (u, v) in order.
constexpr int kRasterBlock = 1024;

__global__ void __launch_bounds__(kRasterBlock) k_slice_counts(StackTab t, unsigned long long *counts) {
  using BR = cub::BlockReduce<int, kRasterBlock>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t s = blockIdx.x;
  const int st = stack_of_slice(t, s);
  const int64_t k = s - t.slice0[st], ns = t.ns[st], npx = t.nx[st] * t.ny[st];
  const uint8_t *m = t.mask[st];
  int c = 0;
  for (int64_t p = threadIdx.x; p < npx; p += kRasterBlock) c += m[p * ns + k] != 0;
  c = BR(tmp).Sum(c);
  if (threadIdx.x == 0) counts[s] = (unsigned long long)c;
}

// motion.py:210-237 (motion.py _stack_points): slice -> raster order, per-slice
// lift with m = the slice's masked count
__global__ void __launch_bounds__(kRasterBlock) k_build_points(StackTab t, const int64_t *__restrict__ slice_off,
                                                               double *__restrict__ x0, int32_t *__restrict__ sid,
                                                               double *__restrict__ vals) {
  using BS = cub::BlockScan<int, kRasterBlock>;
  __shared__ typename BS::TempStorage tmp;
  const int64_t s = blockIdx.x;
  const int st = stack_of_slice(t, s);
  const int64_t k = s - t.slice0[st], ns = t.ns[st], ny = t.ny[st], npx = t.nx[st] * ny;
  const uint8_t *m = t.mask[st];
  const double *d = t.data[st];
  const bool gemv = slice_off[s + 1] - slice_off[s] == 1;
  int64_t base = slice_off[s];
  for (int64_t p0 = 0; p0 < npx; p0 += kRasterBlock) {
    const int64_t p = p0 + threadIdx.x;
    const int f = p < npx && m[p * ns + k] != 0;
    int rank, total;
    BS(tmp).ExclusiveSum(f, rank, total);
    if (f) {
      const int64_t o = base + rank;
      double w[3];
      affine_row(t.A[st], (double)(p / ny), (double)(p % ny), (double)k, gemv, w);
      x0[3 * o] = w[0];
      x0[3 * o + 1] = w[1];
      x0[3 * o + 2] = w[2];
      sid[o] = (int32_t)s;
      vals[o] = d[p * ns + k];
    }
    base += total;
    __syncthreads();  // tmp reuse
  }
}

// ---- content-adaptive sampling ------------------------------------------------
__global__ void k_mask_flags(int64_t n, const uint8_t *__restrict__ m, int32_t *__restrict__ f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    f[i] = m[i] != 0;
}

// initialization.py:44-57 + :95-96 for one stack (C order): the weight
// (1 - lambda) * |grad| + lambda of every masked pixel at its pooled index,
// the pixel's flat index, and (optionally) its value for the 'mean' policy
__global__ void k_init_weights(int64_t nx, int64_t ny, int64_t ns, const double *__restrict__ d,
                               const uint8_t *__restrict__ m, const int32_t *__restrict__ rank, int64_t pool0,
                               double one_minus_lambda, double lambda, double *__restrict__ w,
                               int32_t *__restrict__ flat, double *__restrict__ vals) {
  const int64_t n = nx * ny * ns, su = ny * ns;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    if (!m[i]) continue;
    const int64_t u = i / su, v = (i / ns) % ny;
    double gu, gv;
    if (u == 0) gu = __dsub_rn(d[i + su], d[i]);
    else if (u == nx - 1) gu = __dsub_rn(d[i], d[i - su]);
    else gu = __ddiv_rn(__dsub_rn(d[i + su], d[i - su]), 2.0);
    if (v == 0) gv = __dsub_rn(d[i + ns], d[i]);
    else if (v == ny - 1) gv = __dsub_rn(d[i], d[i - ns]);
    else gv = __ddiv_rn(__dsub_rn(d[i + ns], d[i - ns]), 2.0);
    const int64_t o = pool0 + rank[i];
    w[o] = __dadd_rn(__dmul_rn(one_minus_lambda, glibc_hypot(gu, gv)), lambda);
    flat[o] = (int32_t)i;
    if (vals) vals[o] = d[i];
  }
}

__global__ void k_fill(int64_t n, double v, double *__restrict__ x) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = v;
}

// numpy pairwise_sum (loops_utils.h.src), blocks of <= 128, accumulated in T
// (float64, or float32 for float32 data; inputs are float64 copies, exact)
template <class T>
__device__ __forceinline__ T add_rn(T a, T b);
template <>
__device__ __forceinline__ double add_rn<double>(double a, double b) { return __dadd_rn(a, b); }
template <>
__device__ __forceinline__ float add_rn<float>(float a, float b) { return __fadd_rn(a, b); }

template <class T>
__device__ T pw_block(const double *__restrict__ a, int64_t n) {
  if (n < 8) {
    T r = T(0);
    for (int64_t i = 0; i < n; ++i) r = add_rn<T>(r, (T)a[i]);
    return r;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = (T)a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = add_rn<T>(r[j], (T)a[i + j]);
  }
  T res = add_rn<T>(add_rn<T>(add_rn<T>(r[0], r[1]), add_rn<T>(r[2], r[3])),
                    add_rn<T>(add_rn<T>(r[4], r[5]), add_rn<T>(r[6], r[7])));
  for (; i < n; ++i) res = add_rn<T>(res, (T)a[i]);
  return res;
}

// node `p` at depth `dep` of the pairwise tree over n: its (start, size)
__device__ __forceinline__ void pw_node(int64_t n, int dep, int64_t p, int64_t &start, int64_t &size) {
  start = 0;
  size = n;
  for (int d = 0; d < dep; ++d) {
    int64_t h = size / 2;
    h -= h % 8;
    if ((p >> (dep - 1 - d)) & 1) start += h, size -= h;
    else size = h;
  }
}

// leaves: slot t of 2^D holds the block sum of the node whose leftmost depth-D
// descendant is t (nodes of <= 128 stop descending)
template <class T>
__global__ void k_pw_leaves(int64_t n, int D, const double *__restrict__ a, T *__restrict__ val) {
  const int64_t slots = (int64_t)1 << D;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < slots; t += (int64_t)gridDim.x * blockDim.x) {
    int64_t start = 0, size = n;
    bool own = true;
    for (int d = 0; d < D && size > 128; ++d) {
      int64_t h = size / 2;
      h -= h % 8;
      if ((t >> (D - 1 - d)) & 1) start += h, size -= h;
      else size = h;
      if (size <= 128) own = (t & ((((int64_t)1) << (D - 1 - d)) - 1)) == 0;
    }
    if (own) val[t] = pw_block<T>(a + start, size);
  }
}

// one level of the combine: internal node p at depth dep = left + right
template <class T>
__global__ void k_pw_level(int64_t n, int D, int dep, T *__restrict__ val) {
  const int64_t nodes = (int64_t)1 << dep;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < nodes; p += (int64_t)gridDim.x * blockDim.x) {
    int64_t start, size;
    pw_node(n, dep, p, start, size);
    if (size <= 128) continue;  // a block (its own or an ancestor's leaf slot)
    const int64_t i = p << (D - dep);
    val[i] = add_rn<T>(val[i], val[i + ((int64_t)1 << (D - dep - 1))]);
  }
}

// depth at which every node of the pairwise tree over n is a block (halves are
// not monotone in n -- floor to multiples of 8 -- so the whole tree is walked)
static int pw_depth(int64_t n) {
  if (n <= 128) return 0;
  int64_t h = n / 2;
  h -= h % 8;
  return 1 + std::max(pw_depth(h), pw_depth(n - h));
}

template <class T>
__global__ void k_add0(const T *__restrict__ v, double *__restrict__ out) {
  *out = (double)add_rn<T>(T(0), *v);
}

// numpy np.add.reduce over a (n,) device array (float64 values; accumulated in
// T) -> *out (device scalar, the T result as a double)
template <class T>
static int pairwise_sum(int64_t n, const double *a, double *out, cudaStream_t st) {
  if (n == 0) return fail(GSVR_ERR_INVALID, "pairwise sum of an empty array");
  const int D = pw_depth(n);
  Scratch val;
  GSVR_TRY(val.alloc(sizeof(T) << D, st));
  const int64_t slots = (int64_t)1 << D;
  k_pw_leaves<T><<<grid_for(slots, 128, 148 * 16), 128, 0, st>>>(n, D, a, val.as<T>());
  GSVR_LAUNCH_CHECK("k_pw_leaves");
  for (int dep = D - 1; dep >= 0; --dep) {
    k_pw_level<T><<<grid_for((int64_t)1 << dep, 128, 148 * 16), 128, 0, st>>>(n, D, dep, val.as<T>());
    GSVR_LAUNCH_CHECK("k_pw_level");
  }
  // the reduction's initial value 0 + the tree (umath add reduce)
  k_add0<T><<<1, 1, 0, st>>>(val.as<T>(), out);
  GSVR_LAUNCH_CHECK("k_add0");
  return GSVR_OK;
}

__global__ void k_div_scalar(int64_t n, const double *__restrict__ den, double *__restrict__ x) {
  const double q = *den;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    x[i] = __ddiv_rn(x[i], q);
}

// cumsum (add.accumulate): x[i] = x[i-1] + x[i], in place, one thread.  A ring
// of kChainStages shared-memory chunks: TMA loads run kChainStages-1 chunks
// ahead of the chain, each finished chunk leaves by a TMA bulk store.
// `last` receives x[n-1].  x is padded to an even length (16-byte copies).
constexpr int kChainChunk = 2048;  // doubles (16 KB)
constexpr int kChainStages = 8;

__global__ void __launch_bounds__(32) k_cumsum_chain(int64_t n, double *x, double *last) {
  extern __shared__ __align__(128) unsigned char chain_smem[];
  double *buf = reinterpret_cast<double *>(chain_smem);
  __shared__ __align__(8) uint64_t bar[kChainStages];
  if (threadIdx.x != 0) return;
  const int64_t nch = (n + kChainChunk - 1) / kChainChunk;
  auto chunk_len = [&](int64_t c) { return (int)min((int64_t)kChainChunk, n - c * kChainChunk); };
  auto load = [&](int64_t c) {
    const int len = chunk_len(c), even = (len + 1) & ~1;  // pad element inside the allocation
    tma_load_1d(buf + (c % kChainStages) * kChainChunk, x + c * kChainChunk, (uint32_t)even * 8u,
                &bar[c % kChainStages]);
  };
  for (int s = 0; s < kChainStages; ++s) mbar_init(&bar[s], 1);
  for (int64_t c = 0; c < nch && c < kChainStages; ++c) load(c);
  double acc = 0.0;  // 0.0 + x[0] == x[0] for the non-negative inputs here
  for (int64_t c = 0; c < nch; ++c) {
    const int stg = (int)(c % kChainStages);
    mbar_wait(&bar[stg], (uint32_t)((c / kChainStages) & 1));
    double *b = buf + stg * kChainChunk;
    const int len = chunk_len(c);
    // groups of 8: the next group's shared loads are issued before this
    // group's dependent adds, so only the add latency is exposed
    const int ng = len / 8;
    double2 nx[4];
    if (ng > 0) {
#pragma unroll
      for (int j = 0; j < 4; ++j) nx[j] = reinterpret_cast<const double2 *>(b)[j];
    }
    for (int g = 0; g < ng; ++g) {
      double2 cu[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) cu[j] = nx[j];
      if (g + 1 < ng) {
#pragma unroll
        for (int j = 0; j < 4; ++j) nx[j] = reinterpret_cast<const double2 *>(b + 8 * (g + 1))[j];
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        acc = __dadd_rn(acc, cu[j].x);
        cu[j].x = acc;
        acc = __dadd_rn(acc, cu[j].y);
        cu[j].y = acc;
      }
#pragma unroll
      for (int j = 0; j < 4; ++j) reinterpret_cast<double2 *>(b + 8 * g)[j] = cu[j];
    }
    int i = 8 * ng;
    for (; i < len; ++i) {
      acc = __dadd_rn(acc, b[i]);
      b[i] = acc;
    }
    const int even = len & ~1;
    if (even < len) x[c * kChainChunk + even] = b[even];  // odd tail element
    tma_store_fence();
    if (even > 0) tma_store_1d(x + c * kChainChunk, b, (uint32_t)even * 8u);
    tma_store_commit();
    // the previous chunk's store has read its stage -> refill it
    tma_store_wait_read<1>();
    if (c >= 1 && c - 1 + kChainStages < nch) load(c - 1 + kChainStages);
  }
  tma_store_wait<0>();
  *last = acc;
}

static int cumsum_chain(int64_t n, double *x, double *last, cudaStream_t st) {
  const size_t chain_smem = (size_t)kChainStages * kChainChunk * 8;
  GSVR_TRY(ensure_smem((const void *)k_cumsum_chain, chain_smem));
  k_cumsum_chain<<<1, 32, chain_smem, st>>>(n, x, last);
  GSVR_LAUNCH_CHECK("k_cumsum_chain");
  return GSVR_OK;
}

// side='right' searchsorted of the uniforms in the normalised cdf, then the
// pooled index -> (stack, u, v, k) and the (stack, slice) draw counts
__global__ void k_draw_pixels(int64_t N, const double *__restrict__ u, int64_t P, const double *__restrict__ cdf,
                              const int32_t *__restrict__ flat, StackTab t, int64_t *__restrict__ pix,
                              int *__restrict__ group_count) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    const double x = u[j];
    int64_t lo = 0, hi = P;  // first i with cdf[i] > x
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (cdf[mid] > x) hi = mid;
      else lo = mid + 1;
    }
    const int64_t idx = lo < P ? lo : P - 1;  // x < 1 == cdf[P-1]: never clamps
    int st = 0;  // searchsorted(offs, idx, 'right') - 1
    while (st + 1 < t.n && t.pool0[st + 1] <= idx) ++st;
    const int64_t f = flat[idx];
    const int64_t k = f % t.ns[st];
    pix[j] = ((int64_t)st << 56) | f;
    atomicAdd(group_count + t.slice0[st] + k, 1);
  }
}

__global__ void k_lift_draws(int64_t N, const int64_t *__restrict__ pix, const int *__restrict__ group_count,
                             StackTab t, double *__restrict__ pos) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    const int st = (int)(pix[j] >> 56);
    const int64_t f = pix[j] & ((((int64_t)1) << 56) - 1);
    const int64_t ns = t.ns[st], ny = t.ny[st];
    const int64_t k = f % ns, v = (f / ns) % ny, uu = f / (ns * ny);
    double w[3];
    affine_row(t.A[st], (double)uu, (double)v, (double)k, group_count[t.slice0[st] + k] == 1, w);
    pos[3 * j] = w[0];
    pos[3 * j + 1] = w[1];
    pos[3 * j + 2] = w[2];
  }
}

// ---- initialization.py:109-130: the first stack pixel each position sits on --
__global__ void k_count_nan(int64_t N, const double *__restrict__ c, unsigned long long *cnt) {
  int mine = 0;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x)
    mine += isnan(c[j]) ? 1 : 0;
  mine = __reduce_add_sync(0xffffffffu, mine);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(cnt, (unsigned long long)mine);
}

__global__ void k_source_match(int64_t N, const double *__restrict__ pos, const unsigned long long *__restrict__ todo,
                               int64_t nx, int64_t ny, int64_t ns, const double *__restrict__ d, StackTab inv,
                               int st, double *__restrict__ c) {
  const bool gemv = *todo == 1;
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    if (!isnan(c[j])) continue;
    double idx[3];
    affine_row(inv.A[st], pos[3 * j], pos[3 * j + 1], pos[3 * j + 2], gemv, idx);
    bool ok = true;
    int64_t r[3];
    const int64_t dims[3] = {nx, ny, ns};
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      const double ri = rint(idx[a]);
      ok = ok && fabs(__dsub_rn(idx[a], ri)) < 1e-6;
      r[a] = (int64_t)ri;
      ok = ok && r[a] >= 0 && r[a] < dims[a];
    }
    if (ok) c[j] = d[(r[0] * ny + r[1]) * ns + r[2]];
  }
}

static int make_tab(int n, const gsvr_stack_view *v, StackTab &t) {
  if (n < 1 || n > kMaxStacks) return fail(GSVR_ERR_INVALID, "need 1..%d stacks, got %d", kMaxStacks, n);
  t.n = n;
  t.slice0[0] = 0;
  for (int i = 0; i < n; ++i) {
    if (v[i].nx < 1 || v[i].ny < 1 || v[i].ns < 1) return fail(GSVR_ERR_INVALID, "empty stack");
    if (v[i].nx * v[i].ny * v[i].ns >= ((int64_t)1 << 31)) return fail(GSVR_ERR_INVALID, "stack too large");
    if (!v[i].data || !v[i].mask) return fail(GSVR_ERR_INVALID, "null stack array");
    t.nx[i] = v[i].nx;
    t.ny[i] = v[i].ny;
    t.ns[i] = v[i].ns;
    t.data[i] = v[i].data;
    t.mask[i] = v[i].mask;
    for (int e = 0; e < 12; ++e) t.A[i][e] = v[i].affine[e];
    t.slice0[i + 1] = t.slice0[i] + v[i].ns;
  }
  for (int i = 0; i <= n; ++i) t.pool0[i] = 0;
  return GSVR_OK;
}

// initialization.py:44-57, :95-96 over every stack: pooled weights, flat
// indices and (optionally) values of the masked pixels; t.pool0 filled
static int pooled_weights(const StackTab &t, double lambda_init, double *w, int32_t *flat, double *vals,
                          cudaStream_t st) {
  int64_t maxn = 0;
  for (int i = 0; i < t.n; ++i) maxn = std::max(maxn, t.nx[i] * t.ny[i] * t.ns[i]);
  Scratch rank, scan_tmp;
  GSVR_TRY(rank.alloc(maxn * 4, st));
  size_t tmp_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp_bytes, (int32_t *)nullptr, (int32_t *)nullptr, (int)maxn, st);
  GSVR_TRY(scan_tmp.alloc(tmp_bytes, st));
  const double oml = 1.0 - lambda_init;
  for (int i = 0; i < t.n; ++i) {
    const int64_t n = t.nx[i] * t.ny[i] * t.ns[i];
    k_mask_flags<<<grid_for(n, 256), 256, 0, st>>>(n, t.mask[i], rank.as<int32_t>());
    GSVR_LAUNCH_CHECK("k_mask_flags");
    GSVR_CUDA(cub::DeviceScan::ExclusiveSum(scan_tmp.ptr, tmp_bytes, rank.as<int32_t>(), rank.as<int32_t>(),
                                            (int)n, st));
    k_init_weights<<<grid_for(n, 256), 256, 0, st>>>(t.nx[i], t.ny[i], t.ns[i], t.data[i], t.mask[i],
                                                     rank.as<int32_t>(), t.pool0[i], oml, lambda_init, w, flat,
                                                     vals);
    GSVR_LAUNCH_CHECK("k_init_weights");
  }
  return GSVR_OK;
}

// pooled masked-pixel offsets of each stack from the slice counts
static int64_t fill_pool(StackTab &t, const int64_t *slice_counts) {
  for (int i = 0; i < t.n; ++i) {
    int64_t c = 0;
    for (int64_t s = t.slice0[i]; s < t.slice0[i + 1]; ++s) c += slice_counts[s];
    t.pool0[i + 1] = t.pool0[i] + c;
  }
  return t.pool0[t.n];
}

static int check_grad_shape(const StackTab &t) {
  for (int i = 0; i < t.n; ++i)
    if (t.nx[i] < 2 || t.ny[i] < 2)
      return fail(GSVR_ERR_INVALID,
                  "Shape of array too small to calculate a numerical gradient, at least (edge_order + 1) "
                  "elements are required.");
  return GSVR_OK;
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_stack_slice_counts(int n_stacks, const gsvr_stack_view *stacks, int64_t *counts, void *stream) {
  StackTab t;
  GSVR_TRY(make_tab(n_stacks, stacks, t));
  cudaStream_t st = as_stream(stream);
  const int64_t S = t.slice0[n_stacks];
  Scratch c;
  GSVR_TRY(c.alloc(S * 8, st));
  k_slice_counts<<<(unsigned)S, kRasterBlock, 0, st>>>(t, c.as<unsigned long long>());
  GSVR_LAUNCH_CHECK("k_slice_counts");
  GSVR_CUDA(cudaMemcpyAsync(counts, c.ptr, S * 8, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  return GSVR_OK;
}

int gsvr_build_points(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts, double *x0,
                      int32_t *slice_ids, double *intensities, void *stream) {
  StackTab t;
  GSVR_TRY(make_tab(n_stacks, stacks, t));
  cudaStream_t st = as_stream(stream);
  const int64_t S = t.slice0[n_stacks];
  std::vector<int64_t> off(S + 1, 0);
  for (int64_t s = 0; s < S; ++s) off[s + 1] = off[s] + slice_counts[s];
  if (off[S] == 0) return GSVR_OK;
  if (!x0 || !slice_ids || !intensities) return fail(GSVR_ERR_INVALID, "null output");
  Scratch d;
  GSVR_TRY(d.alloc((S + 1) * 8, st));
  GSVR_CUDA(cudaMemcpyAsync(d.ptr, off.data(), (S + 1) * 8, cudaMemcpyHostToDevice, st));
  k_build_points<<<(unsigned)S, kRasterBlock, 0, st>>>(t, d.as<int64_t>(), x0, slice_ids, intensities);
  GSVR_LAUNCH_CHECK("k_build_points");
  GSVR_CUDA(cudaStreamSynchronize(st));  // `off` is pageable host memory
  return GSVR_OK;
}

int gsvr_init_sample(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts,
                     double lambda_init, int64_t n_draws, const double *uniforms, double *positions,
                     int *uniform_fallback, double *masked_sum, int masked_sum_f32, void *stream) {
  StackTab t;
  GSVR_TRY(make_tab(n_stacks, stacks, t));
  cudaStream_t st = as_stream(stream);
  const int64_t S = t.slice0[n_stacks];
  const int64_t P = fill_pool(t, slice_counts);
  if (P < 1) return fail(GSVR_ERR_INVALID, "no masked pixels to sample from");
  if (P >= ((int64_t)1 << 31)) return fail(GSVR_ERR_INVALID, "too many masked pixels");
  if (n_draws < 0 || (n_draws > 0 && (!uniforms || !positions))) return fail(GSVR_ERR_INVALID, "bad draws");
  GSVR_TRY(check_grad_shape(t));
  Scratch w, flat, vals, scal;
  GSVR_TRY(w.alloc((P + 2) * 8, st));  // + pad for the chain's 16-byte copies
  GSVR_TRY(flat.alloc(P * 4, st));
  if (masked_sum) GSVR_TRY(vals.alloc(P * 8, st));
  GSVR_TRY(scal.alloc(4 * 8, st));  // [0] total, [1] cdf last, [2] masked sum
  GSVR_TRY(pooled_weights(t, lambda_init, w.as<double>(), flat.as<int32_t>(),
                          masked_sum ? vals.as<double>() : nullptr, st));
  double *total = scal.as<double>(), *last = total + 1;
  if (masked_sum) {
    GSVR_TRY(masked_sum_f32 ? pairwise_sum<float>(P, vals.as<double>(), total + 2, st)
                            : pairwise_sum<double>(P, vals.as<double>(), total + 2, st));
    GSVR_CUDA(cudaMemcpyAsync(masked_sum, total + 2, 8, cudaMemcpyDeviceToHost, st));
  }
  // weights.sum() <= 0 -> uniform weights (initialization.py:97-100)
  GSVR_TRY(pairwise_sum<double>(P, w.as<double>(), total, st));
  double h_total = 0.0;
  GSVR_CUDA(cudaMemcpyAsync(&h_total, total, 8, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  *uniform_fallback = !(h_total > 0.0);
  if (*uniform_fallback) {
    k_fill<<<grid_for(P, 256), 256, 0, st>>>(P, 1.0, w.as<double>());
    GSVR_LAUNCH_CHECK("k_fill");
    GSVR_TRY(pairwise_sum<double>(P, w.as<double>(), total, st));
  }
  if (n_draws == 0) return GSVR_OK;
  // prob = weights / total; cdf = prob.cumsum(); cdf /= cdf[-1]
  k_div_scalar<<<grid_for(P, 256), 256, 0, st>>>(P, total, w.as<double>());
  GSVR_LAUNCH_CHECK("k_div_scalar");
  GSVR_TRY(cumsum_chain(P, w.as<double>(), last, st));
  k_div_scalar<<<grid_for(P, 256), 256, 0, st>>>(P, last, w.as<double>());
  GSVR_LAUNCH_CHECK("k_div_scalar");
  Scratch pix, groups;
  GSVR_TRY(pix.alloc(n_draws * 8, st));
  GSVR_TRY(groups.alloc(S * 4, st));
  GSVR_CUDA(cudaMemsetAsync(groups.ptr, 0, S * 4, st));
  k_draw_pixels<<<grid_for(n_draws, 128), 128, 0, st>>>(n_draws, uniforms, P, w.as<double>(), flat.as<int32_t>(), t,
                                                         pix.as<int64_t>(), groups.as<int>());
  GSVR_LAUNCH_CHECK("k_draw_pixels");
  k_lift_draws<<<grid_for(n_draws, 256), 256, 0, st>>>(n_draws, pix.as<int64_t>(), groups.as<int>(), t, positions);
  GSVR_LAUNCH_CHECK("k_lift_draws");
  return GSVR_OK;
}

int gsvr_init_source_intensity(int n_stacks, const gsvr_stack_view *stacks, const double *inv_affines, int64_t N,
                               const double *positions, double *intensities, int64_t *unmatched, void *stream) {
  StackTab t;
  GSVR_TRY(make_tab(n_stacks, stacks, t));
  cudaStream_t st = as_stream(stream);
  for (int i = 0; i < n_stacks; ++i)
    for (int e = 0; e < 12; ++e) t.A[i][e] = inv_affines[16 * i + e];  // inverse affines (host, 4x4 each)
  if (N == 0) {
    *unmatched = 0;
    return GSVR_OK;
  }
  Scratch cnt;
  GSVR_TRY(cnt.alloc((n_stacks + 1) * 8, st));
  GSVR_CUDA(cudaMemsetAsync(cnt.ptr, 0, (n_stacks + 1) * 8, st));
  k_fill<<<grid_for(N, 256), 256, 0, st>>>(N, std::nan(""), intensities);
  GSVR_LAUNCH_CHECK("k_fill");
  unsigned long long *c = cnt.as<unsigned long long>();
  for (int i = 0; i < n_stacks; ++i) {
    k_count_nan<<<grid_for(N, 256), 256, 0, st>>>(N, intensities, c + i);
    GSVR_LAUNCH_CHECK("k_count_nan");
    k_source_match<<<grid_for(N, 256), 256, 0, st>>>(N, positions, c + i, t.nx[i], t.ny[i], t.ns[i], t.data[i], t,
                                                      i, intensities);
    GSVR_LAUNCH_CHECK("k_source_match");
  }
  k_count_nan<<<grid_for(N, 256), 256, 0, st>>>(N, intensities, c + n_stacks);
  GSVR_LAUNCH_CHECK("k_count_nan");
  unsigned long long left = 0;
  GSVR_CUDA(cudaMemcpyAsync(&left, c + n_stacks, 8, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  *unmatched = (int64_t)left;
  return GSVR_OK;
}

int gsvr_init_weights(int n_stacks, const gsvr_stack_view *stacks, const int64_t *slice_counts,
                      double lambda_init, double *weights, void *stream) {
  StackTab t;
  GSVR_TRY(make_tab(n_stacks, stacks, t));
  cudaStream_t st = as_stream(stream);
  const int64_t P = fill_pool(t, slice_counts);
  if (P >= ((int64_t)1 << 31)) return fail(GSVR_ERR_INVALID, "too many masked pixels");
  GSVR_TRY(check_grad_shape(t));
  if (P == 0) return GSVR_OK;
  Scratch flat;
  GSVR_TRY(flat.alloc(P * 4, st));
  GSVR_TRY(pooled_weights(t, lambda_init, weights, flat.as<int32_t>(), nullptr, st));
  return GSVR_OK;
}

int gsvr_cumsum(int64_t n, double *x, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (n == 0) return GSVR_OK;
  Scratch buf, last;
  GSVR_TRY(buf.alloc((n + 2) * 8, st));  // padded copy (the chain reads in 16-byte units)
  GSVR_TRY(last.alloc(8, st));
  GSVR_CUDA(cudaMemcpyAsync(buf.ptr, x, n * 8, cudaMemcpyDeviceToDevice, st));
  GSVR_TRY(cumsum_chain(n, buf.as<double>(), last.as<double>(), st));
  GSVR_CUDA(cudaMemcpyAsync(x, buf.ptr, n * 8, cudaMemcpyDeviceToDevice, st));
  return GSVR_OK;
}

int gsvr_pairwise_sum(int64_t n, const double *x, double *out, void *stream) {
  cudaStream_t st = as_stream(stream);
  Scratch s;
  GSVR_TRY(s.alloc(8, st));
  GSVR_TRY(pairwise_sum<double>(n, x, s.as<double>(), st));
  GSVR_CUDA(cudaMemcpyAsync(out, s.ptr, 8, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  return GSVR_OK;
}

}  // extern "C"
