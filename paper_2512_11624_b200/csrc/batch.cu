// batch.cu -- point batch planning and (slice, tile) binning.
//
// Planning (once per point batch; train.py:373-497 builds the batch once per fit):
//   Morton keys of the nominal positions under the slice id -> device radix sort
//   -> single-slice tiles of <= tile_points consecutive points, balanced per slice
//   -> tile origins (bbox centres, fp64) and fp32 tile-relative offsets.
// Binning (once per neighbour refresh, train.py:462-465): per tile, a segmented
// device radix sort of the tile's P_t*K neighbour ids yields in one pass
//   * the unique-Gaussian list of the tile (ascending ids)        -> gid
//   * the Gaussian-major pair list (pairs of one Gaussian by pixel) -> pair_pix, csr
//   * the pixel-major local ids                                    -> nbr_local
// Counts per (slice, tile) are exact functions of the neighbour lists, so they are
// bit-identical to counts derived from the reference's knn.query output.
#include <cub/block/block_radix_sort.cuh>
#include <cub/block/block_reduce.cuh>
#include <cub/block/block_scan.cuh>
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "batch.cuh"

namespace gsvr {

// ---------------------------------------------------------------------------
// bounding boxes

template <int BLOCK>
__global__ void k_bbox3(const double *__restrict__ p, int64_t n, unsigned long long *keys) {
  using BR = cub::BlockReduce<unsigned long long, BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  for (int64_t i = blockIdx.x * (int64_t)BLOCK + threadIdx.x; i < n; i += (int64_t)gridDim.x * BLOCK) {
    for (int d = 0; d < 3; ++d) {
      unsigned long long k = dkey(p[3 * i + d]);
      lo[d] = k < lo[d] ? k : lo[d];
      hi[d] = k > hi[d] ? k : hi[d];
    }
  }
  for (int d = 0; d < 3; ++d) {
    unsigned long long a = BR(tmp).Reduce(lo[d], cub::Min());
    __syncthreads();
    unsigned long long b = BR(tmp).Reduce(hi[d], cub::Max());
    __syncthreads();
    if (threadIdx.x == 0) {
      atomicMin(&keys[d], a);
      atomicMax(&keys[3 + d], b);
    }
  }
}

__global__ void k_bbox_init(unsigned long long *keys) {
  if (threadIdx.x < 6) keys[threadIdx.x] = threadIdx.x < 3 ? ~0ull : 0ull;
}

// (no host->device copies in the planning path: they would queue behind bulk
// uploads on the copy engine, see gsvr_train_step_backward_host)
int bbox3(const double *pts, int64_t n, unsigned long long *keys_dev, double out[6], cudaStream_t st) {
  k_bbox_init<<<1, 32, 0, st>>>(keys_dev);
  k_bbox3<256><<<grid_for(n, 256, 148 * 4), 256, 0, st>>>(pts, n, keys_dev);
  GSVR_LAUNCH_CHECK("k_bbox3");
  unsigned long long h[6];
  GSVR_CUDA(cudaMemcpyAsync(h, keys_dev, sizeof(h), cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  for (int d = 0; d < 6; ++d) out[d] = dkey_inv(h[d]);
  for (int d = 0; d < 6; ++d)
    if (!std::isfinite(out[d])) return fail(GSVR_ERR_INVALID, "non-finite coordinates");
  return GSVR_OK;
}

// ---------------------------------------------------------------------------
// planning kernels

__global__ void k_morton_keys(int64_t P, const double *__restrict__ x0, const int32_t *__restrict__ sid,
                              int S, double3 lo, double3 inv_ext, int mbits, int sbits,
                              unsigned long long *__restrict__ keys, int32_t *__restrict__ vals,
                              int *bad) {
  const unsigned long long qmax = (1ull << mbits) - 1;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int s = sid[i];
    if (s < 0 || s >= S) { atomicExch(bad, 1); s = 0; }
    double f[3] = {(x0[3 * i] - lo.x) * inv_ext.x, (x0[3 * i + 1] - lo.y) * inv_ext.y,
                   (x0[3 * i + 2] - lo.z) * inv_ext.z};
    unsigned long long code = 0;
    for (int d = 0; d < 3; ++d) {
      double q = f[d] * (double)qmax;
      unsigned long long u = q <= 0.0 ? 0ull : (q >= (double)qmax ? qmax : (unsigned long long)q);
      code |= spread3(u) << (2 - d);
    }
    keys[i] = ((unsigned long long)s << (3 * mbits)) | code;
    vals[i] = (int32_t)i;
    (void)sbits;
  }
}

// Balanced single-slice tiles from the slice counts (one block): slice s of c
// points -> ceil(c/TP) tiles of ~equal size; also the first tile of every slice.
__global__ void __launch_bounds__(1024) k_make_tiles(int64_t S, const unsigned int *__restrict__ counts, int TP,
                             int64_t *__restrict__ ts, int32_t *__restrict__ tn, int32_t *__restrict__ tsl,
                             int32_t *__restrict__ tile0) {
  using BS = cub::BlockScan<long long, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ long long carry_t, carry_p;
  if (threadIdx.x == 0) carry_t = carry_p = 0;
  __syncthreads();
  for (int64_t s0 = 0; s0 < S; s0 += 1024) {
    const int64_t s = s0 + threadIdx.x;
    const long long c = s < S ? (long long)counts[s] : 0;
    const long long nt = (c + TP - 1) / TP;
    long long t_off, p_off, t_tot, p_tot;
    BS(tmp).ExclusiveSum(nt, t_off, t_tot);
    __syncthreads();
    BS(tmp).ExclusiveSum(c, p_off, p_tot);
    const long long tb = carry_t + t_off, pb = carry_p + p_off;
    if (s < S) {
      tile0[s] = (int32_t)tb;
      for (long long i = 0; i < nt; ++i) {
        const long long a = c * i / nt, e = c * (i + 1) / nt;
        ts[tb + i] = pb + a;
        tn[tb + i] = (int32_t)(e - a);
        tsl[tb + i] = (int32_t)s;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry_t += t_tot, carry_p += p_tot;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile0[S] = (int32_t)carry_t;
}

// Per-tile padded segment offsets of nbr_local (16-byte aligned) and pair_pix
// (chunk-blocked) for K neighbours (one block).
__global__ void __launch_bounds__(1024) k_tile_layout(int64_t T, const int32_t *__restrict__ tn, int64_t K, int64_t *__restrict__ nl_off,
                              int64_t *__restrict__ pp_off) {
  using BS = cub::BlockScan<long long, 1024>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ long long ca, cc;
  if (threadIdx.x == 0) ca = cc = 0;
  __syncthreads();
  for (int64_t t0 = 0; t0 < T; t0 += 1024) {
    const int64_t t = t0 + threadIdx.x;
    const long long m = t < T ? (long long)tn[t] * K : 0;
    const long long a = t < T ? (nl_len(tn[t], (int)K) + 7) / 8 * 8 : 0;
    const long long c = t < T ? (long long)chunk_stride((int)m) * kChunkThreads : 0;
    long long ao, at, co, ct;
    BS(tmp).ExclusiveSum(a, ao, at);
    __syncthreads();
    BS(tmp).ExclusiveSum(c, co, ct);
    if (t < T) {
      nl_off[t] = ca + ao;
      pp_off[t] = cc + co;
    }
    __syncthreads();
    if (threadIdx.x == 0) ca += at, cc += ct;
    __syncthreads();
  }
  if (threadIdx.x == 0) nl_off[T] = ca, pp_off[T] = cc;
}

__global__ void k_slice_hist(int64_t P, const int32_t *__restrict__ perm, const int32_t *__restrict__ sid,
                             int32_t *__restrict__ sid_s, unsigned int *__restrict__ counts) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    int s = sid[perm[i]];
    sid_s[i] = s;
    // the points are slice-sorted: a warp almost always sees one slice, so one
    // lane adds the warp's count (no same-address atomic storm)
    const unsigned same = __match_any_sync(__activemask(), s);
    if ((threadIdx.x & 31) == __ffs(same) - 1) atomicAdd(&counts[s], (unsigned)__popc(same));
  }
}

// Cyclic Jacobi eigen-decomposition of a symmetric 3x3 (fp64); columns of V are
// the eigenvectors of the eigenvalues in w.
__device__ inline void jacobi3(double A[3][3], double w[3], double V[3][3]) {
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) V[i][j] = (i == j);
  for (int sweep = 0; sweep < 12; ++sweep) {
    double off = fabs(A[0][1]) + fabs(A[0][2]) + fabs(A[1][2]);
    if (off == 0.0) break;
    for (int p = 0; p < 2; ++p)
      for (int q = p + 1; q < 3; ++q) {
        if (A[p][q] == 0.0) continue;
        const double th = (A[q][q] - A[p][p]) / (2.0 * A[p][q]);
        const double t = (th >= 0 ? 1.0 : -1.0) / (fabs(th) + sqrt(th * th + 1.0));
        const double c = 1.0 / sqrt(t * t + 1.0), s = t * c;
        for (int k = 0; k < 3; ++k) {  // A <- A J
          const double akp = A[k][p], akq = A[k][q];
          A[k][p] = c * akp - s * akq;
          A[k][q] = s * akp + c * akq;
        }
        for (int k = 0; k < 3; ++k) {  // A <- J^T A
          const double apk = A[p][k], aqk = A[q][k];
          A[p][k] = c * apk - s * aqk;
          A[q][k] = s * apk + c * aqk;
        }
        for (int k = 0; k < 3; ++k) {
          const double vkp = V[k][p], vkq = V[k][q];
          V[k][p] = c * vkp - s * vkq;
          V[k][q] = s * vkp + c * vkq;
        }
      }
  }
  for (int i = 0; i < 3; ++i) w[i] = A[i][i];
}

// One CTA per tile: tile origin = centroid (fp64), the tile's plane (principal
// axes of the offsets), then gather/pack points.  nonplanar[0] counts tiles whose
// points leave the plane by more than 1e-8 mm.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_pack_tiles(
    const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn, const int32_t *__restrict__ perm,
    const double *__restrict__ x0, const double *__restrict__ I_obs, double *__restrict__ x0s,
    float4 *__restrict__ d0obs, double *__restrict__ iobs_s, double *__restrict__ origin,
    double *__restrict__ basis, float2 *__restrict__ ab, int *nonplanar, double *__restrict__ radius) {
  using BR = cub::BlockReduce<double, BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  __shared__ double org[3], bas[9];
  const int t = blockIdx.x;
  const int64_t s0 = tstart[t];
  const int n = tn[t];
  // origin = centroid (it lies on the tile's plane; a bbox centre need not)
  for (int d = 0; d < 3; ++d) {
    double acc = 0.0;
    for (int p = threadIdx.x; p < n; p += BLOCK) acc += x0[3 * (int64_t)perm[s0 + p] + d];
    const double tot = BR(tmp).Sum(acc);
    __syncthreads();
    if (threadIdx.x == 0) org[d] = tot / (double)n;
  }
  __syncthreads();
  // second moments of the offsets -> plane axes
  double m6[6] = {0, 0, 0, 0, 0, 0};
  for (int p = threadIdx.x; p < n; p += BLOCK) {
    const int64_t src = perm[s0 + p];
    const double a = x0[3 * src] - org[0], b = x0[3 * src + 1] - org[1], c = x0[3 * src + 2] - org[2];
    m6[0] += a * a; m6[1] += a * b; m6[2] += a * c; m6[3] += b * b; m6[4] += b * c; m6[5] += c * c;
  }
  double mom[6];
  for (int e = 0; e < 6; ++e) {
    mom[e] = BR(tmp).Sum(m6[e]);
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double A[3][3] = {{mom[0], mom[1], mom[2]}, {mom[1], mom[3], mom[4]}, {mom[2], mom[4], mom[5]}};
    double w[3], V[3][3];
    jacobi3(A, w, V);
    int imax = 0, imin = 0;
    for (int i = 1; i < 3; ++i) {
      if (w[i] > w[imax]) imax = i;
      if (w[i] < w[imin]) imin = i;
    }
    if (imax == imin) imin = (imax + 1) % 3;
    double b1[3] = {V[0][imax], V[1][imax], V[2][imax]};
    double nn[3] = {V[0][imin], V[1][imin], V[2][imin]};
    double b2[3] = {nn[1] * b1[2] - nn[2] * b1[1], nn[2] * b1[0] - nn[0] * b1[2], nn[0] * b1[1] - nn[1] * b1[0]};
    double l2 = sqrt(b2[0] * b2[0] + b2[1] * b2[1] + b2[2] * b2[2]);
    for (int d = 0; d < 3; ++d) {
      bas[d] = b1[d];
      bas[3 + d] = b2[d] / l2;
      bas[6 + d] = nn[d];
    }
  }
  __syncthreads();
  if (threadIdx.x < 3) origin[3 * t + threadIdx.x] = org[threadIdx.x];
  if (threadIdx.x < 6) basis[6 * t + threadIdx.x] = bas[threadIdx.x];
  double resid = 0.0, rad = 0.0;
  for (int p = threadIdx.x; p < n; p += BLOCK) {
    const int64_t src = perm[s0 + p];
    double a = x0[3 * src], b = x0[3 * src + 1], c = x0[3 * src + 2];
    x0s[3 * (s0 + p)] = a;
    x0s[3 * (s0 + p) + 1] = b;
    x0s[3 * (s0 + p) + 2] = c;
    const double da = a - org[0], db = b - org[1], dc = c - org[2];
    d0obs[s0 + p] = make_float4((float)da, (float)db, (float)dc, I_obs ? (float)I_obs[src] : 0.f);
    iobs_s[s0 + p] = I_obs ? I_obs[src] : 0.0;
    ab[s0 + p] = make_float2((float)(da * bas[0] + db * bas[1] + dc * bas[2]),
                             (float)(da * bas[3] + db * bas[4] + dc * bas[5]));
    resid = fmax(resid, fabs(da * bas[6] + db * bas[7] + dc * bas[8]));
    rad = fmax(rad, sqrt(da * da + db * db + dc * dc));
  }
  const double rmax = BR(tmp).Reduce(resid, cub::Max());
  if (threadIdx.x == 0 && !(rmax <= 1e-8)) atomicAdd(nonplanar, 1);
  __syncthreads();
  const double radm = BR(tmp).Reduce(rad, cub::Max());
  if (threadIdx.x == 0) radius[t] = radm;
}

__global__ void k_set_observed(int64_t P, const int32_t *__restrict__ perm, const double *__restrict__ I_obs,
                               float4 *__restrict__ d0obs, double *__restrict__ iobs_s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < P; i += (int64_t)gridDim.x * blockDim.x) {
    const double v = I_obs[perm[i]];
    d0obs[i].w = (float)v;
    iobs_s[i] = v;
  }
}

// ---------------------------------------------------------------------------
// binning kernels

// nbr (caller order, P x K, int32/int64) -> nbr_int (internal order) with id checks.
// One warp per point row: coalesced reads of the caller row, coalesced writes.
template <class I>
__global__ void k_gather_nbr(int64_t i0, int64_t i1, int K, int64_t N, const int32_t *__restrict__ perm,
                             const I *__restrict__ nbr, int32_t *__restrict__ out, int *bad) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t i = i0 + ((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5); i < i1; i += warps) {
    const I *src = nbr + (int64_t)perm[i] * K;
    int32_t *dst = out + i * K;
    for (int k = lane; k < K; k += 32) {
      int64_t j = (int64_t)src[k];
      if (j < 0 || j >= N) { atomicExch(bad, 1); j = 0; }
      dst[k] = (int32_t)j;
    }
  }
}

__global__ void k_pair_positions(const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn,
                                 int64_t K, int32_t *__restrict__ vals) {
  const int t = blockIdx.x;
  const int64_t base = tstart[t] * K;
  const int m = tn[t] * (int)K;
  for (int i = threadIdx.x; i < m; i += blockDim.x) vals[base + i] = i;
}

__global__ void k_segment_offsets(int64_t T, const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn,
                                  int64_t K, int64_t *__restrict__ off) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    off[t] = tstart[t] * K;
    if (t == T - 1) off[T] = (tstart[t] + tn[t]) * K;
  }
}

// One CTA per tile over its sorted (id, pair position) segment.
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_bin_tiles(
    const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn, int64_t K,
    const int32_t *__restrict__ skeys, const int32_t *__restrict__ svals,
    const int64_t *__restrict__ nl_off, const int64_t *__restrict__ pp_off,
    uint16_t *__restrict__ nbr_local, uint16_t *__restrict__ pair_pix,
    int32_t *__restrict__ gid_tmp, uint16_t *__restrict__ csr_tmp, int32_t *__restrict__ nuniq,
    uint8_t *__restrict__ rot_flag) {
  using BS = cub::BlockScan<int, BLOCK>;
  __shared__ typename BS::TempStorage tmp;
  __shared__ int carry;
  const int t = blockIdx.x;
  if (threadIdx.x == 0) rot_flag[t] = 1;
  const int64_t base = tstart[t] * K;
  const int n = tn[t];
  const int m = n * (int)K;
  const int C = (m + kChunkThreads - 1) / kChunkThreads;
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int c0 = 0; c0 < m; c0 += BLOCK) {
    const int i = c0 + threadIdx.x;
    int flag = 0, key = 0, val = 0;
    if (i < m) {
      key = skeys[base + i];
      val = svals[base + i];
      flag = (i == 0) || (skeys[base + i - 1] != key);
    }
    int incl, total;
    BS(tmp).InclusiveSum(flag, incl, total);
    const int lid = carry + incl - 1;
    if (i < m) {
      const int p = val / (int)K, k = val - p * (int)K;
      nbr_local[nl_off[t] + nl_index(p, k, n)] = (uint16_t)lid;
      pair_pix[pp_off[t] + pair_slot(i, C)] = (uint16_t)p;
      if (flag) {
        gid_tmp[base + lid] = key;
        csr_tmp[base + lid] = (uint16_t)i;
      }
    }
    __syncthreads();
    if (threadIdx.x == 0) carry += total;
    __syncthreads();
  }
  if (threadIdx.x == 0) nuniq[t] = carry;
}

// One CTA per tile: block radix sort of the tile's (id, pair position) pairs in
// shared memory (stable, so pairs of one Gaussian stay in pixel order), then the
// unique flags / local ids / CSR / pixel-major local ids in the same pass.
constexpr int kBinBlock = 512, kBinItems = 25, kBinCap = kBinBlock * kBinItems;  // 12800 pairs
#ifndef GSVR_BIN_RADIX_BITS
#define GSVR_BIN_RADIX_BITS 6
#endif
using BinSort = cub::BlockRadixSort<uint32_t, kBinBlock, kBinItems, uint16_t, GSVR_BIN_RADIX_BITS>;
using BinScan = cub::BlockScan<int, kBinBlock>;
union BinTemp {
  typename BinSort::TempStorage sort;
  typename BinScan::TempStorage scan;
};
constexpr size_t kBinSmem = sizeof(BinTemp) + kBinCap * sizeof(uint32_t);

__global__ void __launch_bounds__(kBinBlock) k_bin_sort(
    const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn, int K, int bits, int pbits,
    const int64_t *__restrict__ nl_off, const int64_t *__restrict__ pp_off,
    const int32_t *__restrict__ nbr_int, uint16_t *__restrict__ nbr_local, uint16_t *__restrict__ pair_pix,
    int32_t *__restrict__ gid_tmp, uint16_t *__restrict__ csr_tmp, int32_t *__restrict__ nuniq, int t0,
    const int32_t *__restrict__ tile_list, BinSource ext, uint8_t *__restrict__ rot_flag) {
  extern __shared__ unsigned char bin_smem[];
  BinTemp &tmp = *reinterpret_cast<BinTemp *>(bin_smem);
  uint32_t *skeys = reinterpret_cast<uint32_t *>(bin_smem + sizeof(BinTemp));
  const int t = tile_list ? tile_list[blockIdx.x + t0] : blockIdx.x + t0, tid = threadIdx.x;
  if (tid == 0) rot_flag[t] = 1;  // pair runs ascending: k_pair_rotate re-orders them
  const int64_t base = tstart[t] * (int64_t)K;
  const int n = tn[t];
  const int m = n * K;
  const int C = (m + kChunkThreads - 1) / kChunkThreads;
  const uint32_t pbits_pad = (1u << pbits) - 1u;
  uint32_t keys[kBinItems];
  uint16_t vals[kBinItems];
#pragma unroll
  for (int j = 0; j < kBinItems; ++j) {  // blocked arrangement: stable by pair position
    const int i = tid * kBinItems + j;
    uint32_t key = 0xffffffffu;
    if (i < m) {
      if (ext.nbr) {  // caller-order rows read through perm (host-buffer drop-in)
        const int p = i / K;
        const int64_t src = (int64_t)ext.perm[tstart[t] + p] * K + (i - p * K);
        int64_t id = ext.i64 ? reinterpret_cast<const int64_t *>(ext.nbr)[src]
                             : (int64_t)reinterpret_cast<const int32_t *>(ext.nbr)[src];
        if (id < 0 || id >= ext.N) {
          atomicExch(ext.bad, 1);
          id = 0;
        }
        key = (uint32_t)id;
      } else {
        key = (uint32_t)nbr_int[base + i];
      }
    }
    keys[j] = key;
    vals[j] = (uint16_t)i;
  }
  BinSort(tmp.sort).Sort(keys, vals, 0, bits);
#pragma unroll
  for (int j = 0; j < kBinItems; ++j) skeys[tid * kBinItems + j] = keys[j];
  __syncthreads();
  int flags[kBinItems], incl[kBinItems];
#pragma unroll
  for (int j = 0; j < kBinItems; ++j) {
    const int i = tid * kBinItems + j;
    flags[j] = (i < m) && (i == 0 || skeys[i - 1] != keys[j]);
  }
  int total;
  BinScan(tmp.scan).InclusiveSum(flags, incl, total);
  uint32_t pkeys[kBinItems];
  uint16_t lids[kBinItems];
#pragma unroll
  for (int j = 0; j < kBinItems; ++j) {
    const int i = tid * kBinItems + j;
    pkeys[j] = pbits_pad;
    lids[j] = 0;
    if (i < m) {
      const int lid = incl[j] - 1;
      const int v = vals[j];
      const int p = v / K;
      GSVR_DCHECK(p < n && lid < m, "bin_sort pixel/lid", p, lid);
      pair_pix[pp_off[t] + pair_slot(i, C)] = (uint16_t)p;
      if (flags[j]) {
        gid_tmp[base + lid] = (int32_t)keys[j];
        csr_tmp[base + lid] = (uint16_t)i;
      }
      pkeys[j] = (uint32_t)p;
      lids[j] = (uint16_t)lid;
    }
  }
  __syncthreads();
  // second stable sort by pixel: each pixel's K local ids in ascending order, so
  // lanes (adjacent pixels) of the forward gather nearby records at every k
  // (distance order measured 15% slower in the tile kernel)
  BinSort(tmp.sort).Sort(pkeys, lids, 0, pbits);
#pragma unroll
  for (int j = 0; j < kBinItems; ++j) {
    const int i = tid * kBinItems + j;
    if (i < m) {
      const int p = i / K, k = i - p * K;
      nbr_local[nl_off[t] + nl_index(p, k, n)] = lids[j];
    }
  }
  if (tid == 0) nuniq[t] = total;
}

// ---- hash + bitmask binning (replaces the two block sorts) ---------------
// One CTA per tile.  The tile's neighbour ids go into a shared hash set; the
// unique ids are ranked (ascending id -> local id, as the sorted path); a
// 256-bit pixel mask per local Gaussian records which pixels list it.  From the
// masks: pair counts (CSR), each Gaussian's pixel list in ascending pixel order
// (pair_pix) and each pixel's local ids in ascending order (nbr_local) -- the
// same outputs as k_bin_sort, bit for bit, without sorting the 12,800 pairs.
// Tiles with more than kHashU unique Gaussians are listed for k_bin_sort.
constexpr int kHashBlock = 512, kHashSlots = 4096, kHashU = 1024;
constexpr size_t kHashSmem = kHashSlots * 4 + kHashSlots * 2 + kHashU * 4 * 2 + kHashU * 32 + (kHashU + 1) * 4;

__device__ inline uint32_t hash_slot(uint32_t x) {
  x ^= x >> 16;
  x *= 0x7feb352dU;
  x ^= x >> 15;
  x *= 0x846ca68bU;
  x ^= x >> 16;
  return x & (kHashSlots - 1);
}

// Backward pair order (bank-aware): inside each (tile, Gaussian) run the
// pixels are emitted so that the pair a thread reads at step j of its chunk c
// has pixel id = (j + c) mod 8 whenever the run still holds such a pixel (else
// the lowest pixel of the next non-empty class after it).  The tile kernel's backward fetches one 16-byte
// pixel entry per pair and the 8 lanes of a shared-memory phase are 8
// consecutive chunks, so their bank groups become distinct (ascending runs put
// ~2.5 lanes on the busiest group).  Any order is valid -- a run's moments are
// sums over it -- and the rule is deterministic.  The hash binning emits this
// order directly (k_bin_hash step 6); tiles binned by a sorting path are
// re-ordered here, after compaction (runs holding a repeated pixel keep the
// ascending order).
// The run's pixels as 8 residue classes: bit k of cls[q * stride] = pixel 8k + q.
// Takes the lowest pixel of class `want`, else of the next non-empty class.
#ifndef GSVR_ROT_FULLEST  // GSVR_ROT_FULLEST: the round-2a rule (fullest class), A/B only
__device__ inline int rot_pick(uint32_t *cls, int stride, int want) {
  int q = want;
  uint32_t b = cls[q * stride];
  for (int s = 1; !b && s < 8; ++s) q = (want + s) & 7, b = cls[q * stride];
  cls[q * stride] = b & (b - 1);
  return 8 * (__ffs(b) - 1) + q;
}
// Same rule with the non-empty classes as bits of a register (nz)
__device__ inline int rot_pick_nz(uint32_t *cls, int stride, int want, uint32_t &nz) {
  int q = want;
  if (!((nz >> want) & 1u)) q = (want + __ffs(((nz | (nz << 8)) >> (want + 1)) & 0xffu)) & 7;
  const uint32_t b = cls[q * stride], rest = b & (b - 1);
  cls[q * stride] = rest;
  if (!rest) nz &= ~(1u << q);
  return 8 * (__ffs(b) - 1) + q;
}
#else
__device__ inline int rot_pick(uint32_t *cls, int stride, int want) {
  int q = want;
  uint32_t b = cls[q * stride];
  if (!b) {  // class exhausted: draw from the fullest class (keeps the rest balanced)
    int best = -1;
#pragma unroll
    for (int s = 1; s < 8; ++s) {
      const int qq = (want + s) & 7;
      const uint32_t bb = cls[qq * stride];
      const int c = __popc(bb);
      if (c > best) best = c, q = qq, b = bb;
    }
  }
  cls[q * stride] = b & (b - 1);
  return 8 * (__ffs(b) - 1) + q;
}
// Same rule with the 8 class sizes in a packed register (6 bits each, <= 32):
// the fullest-class search runs on registers, ties to the first class after
// `want` as above.  cnt is updated with the pick.
__device__ inline int rot_pick_counted(uint32_t *cls, int stride, int want, uint64_t &cnt) {
  int q = want;
  if (((cnt >> (6 * q)) & 63u) == 0) {
    int best = -1;
#pragma unroll
    for (int s = 1; s < 8; ++s) {
      const int qq = (want + s) & 7;
      const int c = (int)((cnt >> (6 * qq)) & 63u);
      if (c > best) best = c, q = qq;
    }
  }
  const uint32_t b = cls[q * stride];
  cls[q * stride] = b & (b - 1);
  cnt -= 1ull << (6 * q);
  return 8 * (__ffs(b) - 1) + q;
}
#endif

__global__ void __launch_bounds__(256) k_pair_rotate(const int32_t *__restrict__ tn, int K,
                                                     const int32_t *__restrict__ uoff,
                                                     const uint16_t *__restrict__ csr,
                                                     const int64_t *__restrict__ pp_off,
                                                     const uint8_t *__restrict__ flag,
                                                     uint16_t *__restrict__ pair_pix) {
  __shared__ uint32_t cls_s[8 * 256];
  const int t = blockIdx.x, tid = threadIdx.x;
  if (!flag[t]) return;
  const int m = tn[t] * K, C = chunk_len(m);
  const int u0 = uoff[t], nU = uoff[t + 1] - u0;
  const uint16_t *cs = csr + u0 + t;
  uint16_t *pp = pair_pix + pp_off[t];
  uint32_t *cls = cls_s + tid;
  auto slot = [&](int c, int r) { return ((int64_t)(r >> 3) * kChunkThreads + c) * 8 + (r & 7); };
  for (int l = tid; l < nU; l += blockDim.x) {
    const int i0 = cs[l], i1 = cs[l + 1];
    for (int q = 0; q < 8; ++q) cls[q * 256] = 0u;
    bool dup = false;
    int c = i0 / C, r = i0 - c * C;
    for (int i = i0; i < i1; ++i) {
      const int p = pp[slot(c, r)];
      const uint32_t bit = 1u << (p >> 3);
      dup |= (cls[(p & 7) * 256] & bit) != 0u;
      cls[(p & 7) * 256] |= bit;
      if (++r == C) r = 0, ++c;
    }
    if (dup) continue;  // a repeated pixel: keep the ascending run
    c = i0 / C, r = i0 - c * C;
    for (int i = i0; i < i1; ++i) {
      pp[slot(c, r)] = (uint16_t)rot_pick(cls, 256, (r + c) & 7);
      if (++r == C) r = 0, ++c;
    }
  }
}

// GSVR_PAIR_ROTATE=0 keeps each run's pixels ascending (A/B)
static bool pair_rotate_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_PAIR_ROTATE");
    return !(v && v[0] == '0');
  }();
  return on;
}

#ifdef GSVR_BIN_PROFILE
// diagnostics build only: per-phase block cycles of k_bin_hash (thread 0, between barriers)
__device__ unsigned long long g_bin_phase[10];
#define BIN_PH(i)                                                          \
  if (tid == 0) {                                                          \
    const long long now_ = clock64();                                      \
    atomicAdd(&g_bin_phase[i], (unsigned long long)(now_ - tp_));          \
    tp_ = now_;                                                            \
  }
#define BIN_SYNC() __syncthreads()
#else
#define BIN_PH(i)
#define BIN_SYNC()
#endif

__global__ void __launch_bounds__(kHashBlock) k_bin_hash(
    const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn, int K,
    const int64_t *__restrict__ nl_off, const int64_t *__restrict__ pp_off,
    const int32_t *__restrict__ nbr_int, uint16_t *__restrict__ nbr_local, uint16_t *__restrict__ pair_pix,
    int32_t *__restrict__ gid_tmp, uint16_t *__restrict__ csr_tmp, int32_t *__restrict__ nuniq, int t0,
    const int32_t *__restrict__ tile_list, BinSource ext, int32_t *__restrict__ overflow,
    int *__restrict__ n_overflow, int rot) {
  extern __shared__ __align__(16) unsigned char hash_smem[];
  uint32_t *hkey = reinterpret_cast<uint32_t *>(hash_smem);                // [kHashSlots]
  uint16_t *hlid = reinterpret_cast<uint16_t *>(hkey + kHashSlots);        // [kHashSlots]
  uint32_t *ugid = reinterpret_cast<uint32_t *>(hlid + kHashSlots);        // [kHashU] unique ids (slot order)
  uint32_t *uslot = ugid + kHashU;                                         // [kHashU]
  uint32_t *mask = uslot + kHashU;                                         // [kHashU][8]
  int32_t *csr = reinterpret_cast<int32_t *>(mask + kHashU * 8);           // [kHashU + 1]
  __shared__ int n_unique, too_many;
  using Scan = cub::BlockScan<int, kHashBlock>;
  __shared__ typename Scan::TempStorage scan_tmp;

  const int t = tile_list ? tile_list[blockIdx.x + t0] : blockIdx.x + t0, tid = threadIdx.x;
  const int64_t base = tstart[t] * (int64_t)K;
  const int n = tn[t];
  const int m = n * K;
  const int C = chunk_len(m);
  const uint64_t mK = div_magic(K);  // m * K <= 65535 * K: exact
  auto pair_id = [&](int i) -> uint32_t {
    if (ext.nbr) {  // caller-order rows through perm (host-buffer drop-in)
      const int p = div_by(i, mK);
      const int64_t src = (int64_t)ext.perm[tstart[t] + p] * K + (i - p * K);
      int64_t id = ext.i64 ? reinterpret_cast<const int64_t *>(ext.nbr)[src]
                           : (int64_t)reinterpret_cast<const int32_t *>(ext.nbr)[src];
      if (id < 0 || id >= ext.N) {
        atomicExch(ext.bad, 1);
        id = 0;
      }
      return (uint32_t)id;
    }
    return (uint32_t)nbr_int[base + i];
  };
#ifdef GSVR_BIN_PROFILE
  long long tp_ = clock64();
#endif
  for (int h = tid; h < kHashSlots; h += kHashBlock) hkey[h] = 0xffffffffu;
  if (tid == 0) too_many = 0;
  __syncthreads();
  BIN_PH(0);
  // 1. unique ids into the hash set (a full table hands the tile to the sort);
  // ids fetched four strides ahead of their insertion (independent loads in flight)
  constexpr int kAhead = 4;
  for (int i0 = tid; i0 < m; i0 += kAhead * kHashBlock) {
    uint32_t gg[kAhead];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) gg[u] = i0 + u * kHashBlock < m ? pair_id(i0 + u * kHashBlock) : 0xffffffffu;
#pragma unroll 1
    for (int u = 0; u < kAhead; ++u) {
    const uint32_t g = gg[u];
    if (g == 0xffffffffu) break;
    uint32_t h = hash_slot(g);
    int probes = 0;
    for (;;) {
      // most inserts repeat an id already present (~230 unique of 12,800 per
      // tile): a plain read settles them without an atomic on a hot slot
      const uint32_t cur = *(volatile uint32_t *)&hkey[h];
      if (cur == g) break;
      if (cur == 0xffffffffu) {
        const uint32_t old = atomicCAS(&hkey[h], 0xffffffffu, g);
        if (old == 0xffffffffu || old == g) break;
      }
      h = (h + 1) & (kHashSlots - 1);
      if (++probes >= kHashSlots) {
        too_many = 1;
        break;
      }
    }
    }
  }
  __syncthreads();
  BIN_PH(1);
  // 2. compact the occupied slots
  {
    constexpr int per = kHashSlots / kHashBlock;
    int f[per], pos[per];
#pragma unroll
    for (int j = 0; j < per; ++j) f[j] = hkey[tid * per + j] != 0xffffffffu;
    int total;
    Scan(scan_tmp).ExclusiveSum(f, pos, total);
    if (tid == 0) n_unique = total;
    if (total <= kHashU) {
#pragma unroll
      for (int j = 0; j < per; ++j)
        if (f[j]) ugid[pos[j]] = hkey[tid * per + j], uslot[pos[j]] = tid * per + j;
    }
  }
  __syncthreads();
  BIN_PH(2);
  const int nU = n_unique;
  if (nU > kHashU || too_many) {  // too many for the masks: the sorting kernel takes this tile
    if (tid == 0) {
      overflow[atomicAdd(n_overflow, 1)] = t;
      nuniq[t] = 0;
    }
    return;
  }
  // 3. local id = rank of the id among the tile's unique ids (ascending)
  for (int j = tid; j < nU; j += kHashBlock) {
    const uint32_t g = ugid[j];
    int r = 0;
    for (int k = 0; k < nU; ++k) r += ugid[k] < g;
    hlid[uslot[j]] = (uint16_t)r;
    gid_tmp[base + r] = (int32_t)g;
  }
  for (int w = tid; w < nU * 8; w += kHashBlock) mask[w] = 0u;
  __syncthreads();
  BIN_PH(3);
  // 4. pixel masks
  for (int i0 = tid; i0 < m; i0 += kAhead * kHashBlock) {
    uint32_t gg[kAhead];
#pragma unroll
    for (int u = 0; u < kAhead; ++u) gg[u] = i0 + u * kHashBlock < m ? pair_id(i0 + u * kHashBlock) : 0xffffffffu;
#pragma unroll
    for (int u = 0; u < kAhead; ++u) {
      const int i = i0 + u * kHashBlock;
      if (i >= m) break;
      const uint32_t g = gg[u];
      uint32_t h = hash_slot(g);
      while (hkey[h] != g) h = (h + 1) & (kHashSlots - 1);
      const int p = div_by(i, mK);
      // residue-class layout: word q of a Gaussian holds pixels 8k + q as bit k
      atomicOr(&mask[hlid[h] * 8 + (p & 7)], 1u << (p >> 3));
    }
  }
  __syncthreads();
  BIN_PH(4);
  // 5. pair counts -> CSR (pairs of one Gaussian contiguous, Gaussians ascending)
  {
    constexpr int per = kHashU / kHashBlock;
    int cnt[per], pos[per];
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int l = tid * per + j;
      int c = 0;
      if (l < nU)
#pragma unroll
        for (int w = 0; w < 8; ++w) c += __popc(mask[l * 8 + w]);
      cnt[j] = c;
    }
    int total;
    Scan(scan_tmp).ExclusiveSum(cnt, pos, total);
#pragma unroll
    for (int j = 0; j < per; ++j) {
      const int l = tid * per + j;
      if (l < nU) {
        csr[l] = pos[j];
        csr_tmp[base + l] = (uint16_t)pos[j];
      }
    }
    if (tid == 0) {
      csr[nU] = total;
      too_many = total != m;  // an id repeated within a pixel's row: only the sort keeps both pairs
    }
  }
  __syncthreads();
  BIN_PH(5);
  if (too_many) {
    if (tid == 0) {
      overflow[atomicAdd(n_overflow, 1)] = t;
      nuniq[t] = 0;
    }
    return;
  }
  // 6. Gaussian-major pair list, pair_slot(i, C) stepped incrementally (chunk
  // c, position r inside it): each Gaussian's pixels ascending, or in the
  // bank-aware rotated order (k_pair_rotate's rule; the residue classes live
  // in the hash table's storage, dead after step 4)
  for (int l = tid; l < nU; l += kHashBlock) {
    const int i0 = csr[l], i1 = csr[l + 1];
    int c = i0 / C, r = i0 - c * C;
    uint16_t *pp = pair_pix + pp_off[t];
    if (rot) {
      uint32_t *cls = hkey + tid;
#ifndef GSVR_ROT_FULLEST
      uint32_t nz = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t w = mask[l * 8 + q];
        cls[q * kHashBlock] = w;
        nz |= (w != 0u ? 1u : 0u) << q;
      }
#else
      uint64_t cnt = 0;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t w = mask[l * 8 + q];
        cls[q * kHashBlock] = w;
        cnt |= (uint64_t)__popc(w) << (6 * q);
      }
#endif
      int slot = ((r >> 3) * kChunkThreads + c) * 8 + (r & 7);  // pair_slot, stepped
      for (int i = i0; i < i1; ++i) {
#ifndef GSVR_ROT_FULLEST
        pp[slot] = (uint16_t)rot_pick_nz(cls, kHashBlock, (r + c) & 7, nz);
#else
        pp[slot] = (uint16_t)rot_pick_counted(cls, kHashBlock, (r + c) & 7, cnt);
#endif
        if (++r == C) r = 0, ++c, slot = c * 8;
        else slot += (r & 7) ? 1 : kChunkThreads * 8 - 7;
      }
    } else {  // ascending (A/B only)
#pragma unroll 1
      for (int p = 0; p < n; ++p)
        if ((mask[l * 8 + (p & 7)] >> (p >> 3)) & 1u) {
          pp[((int64_t)(r >> 3) * kChunkThreads + c) * 8 + (r & 7)] = (uint16_t)p;
          if (++r == C) r = 0, ++c;
        }
    }
  }
  BIN_SYNC();
  BIN_PH(6);
  // 7. pixel-major local ids, ascending per pixel.  The Gaussian-major masks
  // are transposed 32 x 32 bits at a time by warp shuffles into per-pixel
  // bitmaps over the local ids (in the hash set's dead hlid/ugid/uslot
  // storage), whose set bits are then the pixel's ids in ascending order.
  const int W = (nU + 31) >> 5, Ws = W | 1;  // odd stride: conflict-free per-pixel reads
  if (W <= 15) {  // (hlid.. are free since step 4; step 6 touches only hkey, mask, csr)
    uint32_t *pix = reinterpret_cast<uint32_t *>(hlid);
    const int warp = tid >> 5, lane = tid & 31;
    for (int task = warp; task < W * 8; task += kHashBlock / 32) {
      const int j = task >> 3, q = task & 7, l = 32 * j + lane;
      uint32_t x = l < nU ? mask[l * 8 + q] : 0u;  // row l: bit k = pixel 8k + q
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const uint32_t m = o == 16 ? 0x0000ffffu : o == 8 ? 0x00ff00ffu : o == 4 ? 0x0f0f0f0fu
                         : o == 2 ? 0x33333333u : 0x55555555u;
        const uint32_t y = __shfl_xor_sync(0xffffffffu, x, o);
        x = (lane & o) ? ((x & ~m) | ((y >> o) & m)) : ((x & m) | ((y & m) << o));
      }
      const int p = 8 * lane + q;  // lane k now holds pixel 8k + q: bit l' = Gaussian 32 j + l'
      if (p < n) pix[p * Ws + j] = x;
    }
    __syncthreads();
    BIN_PH(7);
    if (tid < n) {  // every pixel holds exactly K ids (step 5): a uniform K-step loop,
      const int p = tid;  // only the skip over empty words diverges
      int w = 0;
      uint32_t word = pix[p * Ws];
      for (int k = 0; k < K; ++k) {
        while (word == 0u) word = pix[p * Ws + (++w)];
        const int b = __ffs(word) - 1;
        word &= word - 1;
        nbr_local[nl_off[t] + nl_index(p, k, n)] = (uint16_t)(32 * w + b);
      }
    }
  } else if (tid < n) {
    const int p = tid;
    const int w = p & 7;
    const uint32_t bit = 1u << (p >> 3);
    int k = 0;
    for (int l = 0; l < nU; ++l)
      if (mask[l * 8 + w] & bit) nbr_local[nl_off[t] + nl_index(p, k++, n)] = (uint16_t)l;
  }
  BIN_SYNC();
  BIN_PH(8);
  if (tid == 0) nuniq[t] = nU;
}

__global__ void k_compact_unique(const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn, int64_t K,
                                 const int32_t *__restrict__ uoff, const int32_t *__restrict__ gid_tmp,
                                 const uint16_t *__restrict__ csr_tmp, int32_t *__restrict__ gid,
                                 uint16_t *__restrict__ csr) {
  const int t = blockIdx.x;
  const int64_t base = tstart[t] * K;
  const int u0 = uoff[t], nu = uoff[t + 1] - u0;
  for (int g = threadIdx.x; g < nu; g += blockDim.x) {
    gid[u0 + g] = gid_tmp[base + g];
    csr[u0 + t + g] = csr_tmp[base + g];
  }
  if (threadIdx.x == 0) csr[u0 + t + nu] = (uint16_t)(tn[t] * (int)K);
}

// key = position of Gaussian j's first record (U when it has none), value = j
__global__ void k_first_record(int64_t N, const int32_t *__restrict__ ptr, const int32_t *__restrict__ idx,
                               uint32_t *__restrict__ key, int32_t *__restrict__ val) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    const int a = ptr[j], e = ptr[j + 1];
    key[j] = a < e ? (uint32_t)idx[a] : 0x7fffffffu;
    val[j] = (int32_t)j;
  }
}

__global__ void k_iota(int64_t n, int32_t *out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int32_t)i;
}

// ptr[j] = first position of key j in the sorted keys (j = 0..N).
__global__ void k_lower_bounds(int64_t N, int64_t U, const int32_t *__restrict__ skeys, int32_t *__restrict__ ptr) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= N; j += (int64_t)gridDim.x * blockDim.x) {
    int64_t lo = 0, hi = U;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (skeys[mid] < j) lo = mid + 1; else hi = mid;
    }
    ptr[j] = (int32_t)lo;
  }
}

// dfield[j] += sum over j's records in tile order (deterministic).
// dfield[j] += sum of Gaussian j's (tile, Gaussian) partials: four lanes per
// Gaussian, lane q takes records q, q+4, ... (in tile order), then a fixed
// two-step shuffle tree -> deterministic; the record loads of a Gaussian overlap.
__global__ void __launch_bounds__(256) k_gather_grads(int64_t N, const int32_t *__restrict__ ptr,
                                                      const int32_t *__restrict__ idx,
                                                      const int32_t *__restrict__ order,
                                                      const float *__restrict__ gpart, float *__restrict__ dfield) {
  const int q = threadIdx.x & 3;
  const int64_t groups = (int64_t)gridDim.x * (blockDim.x >> 2);
  for (int64_t jj = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 2;; jj += groups) {
    const bool live = jj < N;
    const int64_t j = live ? order[jj] : 0;
    if (!__any_sync(0xffffffffu, live)) break;  // warp-uniform exit (shuffles below)
    float acc[10];
#pragma unroll
    for (int e = 0; e < 10; ++e) acc[e] = 0.f;
    if (live) {
      const int k1 = ptr[j + 1];
      for (int k = ptr[j] + q; k < k1; k += 4) {
        // a 40-byte record is 16-byte aligned at even u, 8 bytes past at odd u:
        // three loads either way (float4 float4 float2 / float2 float4 float4)
        const int64_t u = idx[k];
        const float *r = gpart + 10 * u;
        float v[10];
        if ((u & 1) == 0) {
          const float4 a = *reinterpret_cast<const float4 *>(r), b = *reinterpret_cast<const float4 *>(r + 4);
          const float2 c = *reinterpret_cast<const float2 *>(r + 8);
          v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
          v[8] = c.x; v[9] = c.y;
        } else {
          const float2 a = *reinterpret_cast<const float2 *>(r);
          const float4 b = *reinterpret_cast<const float4 *>(r + 2), c = *reinterpret_cast<const float4 *>(r + 6);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y; v[4] = b.z; v[5] = b.w; v[6] = c.x; v[7] = c.y;
          v[8] = c.z; v[9] = c.w;
        }
#pragma unroll
        for (int e = 0; e < 10; ++e) acc[e] += v[e];
      }
    }
#pragma unroll
    for (int e = 0; e < 10; ++e) {
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 1);
      acc[e] += __shfl_xor_sync(0xffffffffu, acc[e], 2);
    }
    if (live) {
      float *d = dfield + 10 * j;
#pragma unroll
      for (int e = 0; e < 10; ++e)
        if ((e & 3) == q) d[e] += acc[e];
    }
  }
}

// dslice[s] += sum of slice s's per-tile partials: one block per slice, thread
// i takes tiles i, i+256, ...; fixed block tree -> deterministic.
__global__ void __launch_bounds__(256) k_slice_reduce(int64_t S, const int32_t *__restrict__ tile0,
                                                      const double *__restrict__ tpart,
                                                      double *__restrict__ dslice) {
  using BR = cub::BlockReduce<double, 256>;
  __shared__ typename BR::TempStorage tmp;
  const int64_t s = blockIdx.x;
  double acc[20];
#pragma unroll
  for (int e = 0; e < 20; ++e) acc[e] = 0.0;
  for (int t = tile0[s] + threadIdx.x; t < tile0[s + 1]; t += 256) {
    const double2 *r = reinterpret_cast<const double2 *>(tpart + 20 * (int64_t)t);
#pragma unroll
    for (int e = 0; e < 10; ++e) {
      const double2 v = r[e];
      acc[2 * e] += v.x;
      acc[2 * e + 1] += v.y;
    }
  }
#pragma unroll
  for (int e = 0; e < 20; ++e) {
    const double tot = BR(tmp).Sum(acc[e]);
    if (threadIdx.x == 0) dslice[20 * s + e] += tot;
    __syncthreads();
  }
}

int gather_grads(const gsvr_batch *b, float *dfield, double *dslice, cudaStream_t st) {
  k_gather_grads<<<grid_for(b->N * 4, 256, 148 * 16), 256, 0, st>>>(b->N, b->jr_ptr, b->jr_idx, b->gorder,
                                                                    b->gpart, dfield);
  GSVR_LAUNCH_CHECK("k_gather_grads");
  k_slice_reduce<<<(unsigned)b->S, 256, 0, st>>>(b->S, b->slice_tile0, b->tpart, dslice);
  GSVR_LAUNCH_CHECK("k_slice_reduce");
  return GSVR_OK;
}

__global__ void k_scatter_nbr(int64_t P, int64_t K, const int32_t *__restrict__ perm,
                              const int32_t *__restrict__ nbr_int, int64_t *__restrict__ out) {
  const int64_t total = P * K;
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = e / K, k = e - i * K;
    out[(int64_t)perm[i] * K + k] = nbr_int[e];
  }
}

// ---------------------------------------------------------------------------

int batch_create(int64_t P, int64_t S, const double *x0, const int32_t *sid, const double *I_obs,
                 int tile_points, gsvr_batch **out, cudaStream_t st) {
  *out = nullptr;
  if (P < 1 || S < 1) return fail(GSVR_ERR_INVALID, "empty point batch");
  if (P > INT32_MAX) return fail(GSVR_ERR_INVALID, "too many points for one batch");
  if (tile_points < 1 || tile_points > 1024) return fail(GSVR_ERR_INVALID, "tile_points must be in [1, 1024]");
  gsvr_batch *b = new gsvr_batch();
  b->P = P;
  b->S = S;
  b->TP = tile_points;
  b->owner_stream = st;
  auto bail = [&](int rc) { delete b; return rc; };

  Scratch keys_bb, keys, keys2, vals, tmp, flag, counts;
  if (int rc = keys_bb.alloc(6 * sizeof(unsigned long long), st)) return bail(rc);
  double bb[6];
  if (int rc = bbox3(x0, P, keys_bb.as<unsigned long long>(), bb, st)) return bail(rc);
  int sbits = 1;
  while ((1ll << sbits) < S) ++sbits;
  int mbits = std::min(21, (64 - sbits) / 3);
  double3 lo = make_double3(bb[0], bb[1], bb[2]);
  double ext[3] = {bb[3] - bb[0], bb[4] - bb[1], bb[5] - bb[2]};
  double3 inv = make_double3(ext[0] > 0 ? 1.0 / ext[0] : 0.0, ext[1] > 0 ? 1.0 / ext[1] : 0.0,
                             ext[2] > 0 ? 1.0 / ext[2] : 0.0);

  if (int rc = keys.alloc(P * 8, st)) return bail(rc);
  if (int rc = keys2.alloc(P * 8, st)) return bail(rc);
  if (int rc = vals.alloc(P * 4, st)) return bail(rc);
  if (int rc = flag.alloc(4, st)) return bail(rc);
  if (cudaMemsetAsync(flag.ptr, 0, 4, st) != cudaSuccess) return bail(cuda_status(cudaGetLastError(), "memset"));
  cudaMallocAsync((void **)&b->perm, P * 4, st);
  k_morton_keys<<<grid_for(P, 256), 256, 0, st>>>(P, x0, sid, (int)S, lo, inv, mbits, sbits,
                                                  keys.as<unsigned long long>(), vals.as<int32_t>(),
                                                  flag.as<int>());
  size_t tbytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, tbytes, keys.as<unsigned long long>(), keys2.as<unsigned long long>(),
                                  vals.as<int32_t>(), b->perm, (int)P, 0, 3 * mbits + sbits, st);
  if (int rc = tmp.alloc(tbytes, st)) return bail(rc);
  cub::DeviceRadixSort::SortPairs(tmp.ptr, tbytes, keys.as<unsigned long long>(), keys2.as<unsigned long long>(),
                                  vals.as<int32_t>(), b->perm, (int)P, 0, 3 * mbits + sbits, st);
  if (cudaGetLastError() != cudaSuccess) return bail(fail(GSVR_ERR_CUDA, "radix sort failed"));

  if (int rc = counts.alloc(S * 4, st)) return bail(rc);
  cudaMemsetAsync(counts.ptr, 0, S * 4, st);
  cudaMallocAsync((void **)&b->sid_s, P * 4, st);
  k_slice_hist<<<grid_for(P, 256), 256, 0, st>>>(P, b->perm, sid, b->sid_s, counts.as<unsigned int>());
  std::vector<unsigned int> hc(S);
  int hbad = 0;
  cudaMemcpyAsync(hc.data(), counts.ptr, S * 4, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&hbad, flag.ptr, 4, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return bail(cuda_status(cudaGetLastError(), "planning"));
  if (hbad) return bail(fail(GSVR_ERR_INVALID, "slice id out of range [0, %lld)", (long long)S));

  // Balanced single-slice tiles: a slice of c points -> ceil(c/TP) tiles of ~equal size
  // (built on the device; the host keeps copies of starts and sizes)
  int64_t T = 0;
  for (int64_t s = 0; s < S; ++s) T += (hc[s] + tile_points - 1) / tile_points;
  b->T = T;
  cudaMallocAsync((void **)&b->tpart, (b->T + 1) * 160, st);
  cudaMallocAsync((void **)&b->slice_tile0, (S + 1) * 4, st);
  cudaMallocAsync((void **)&b->tile_start, b->T * 8, st);
  cudaMallocAsync((void **)&b->tile_n, b->T * 4, st);
  cudaMallocAsync((void **)&b->tile_slice, b->T * 4, st);
  cudaMallocAsync((void **)&b->tile_origin, b->T * 24, st);
  cudaMallocAsync((void **)&b->tile_radius, b->T * 8, st);
  cudaMallocAsync((void **)&b->x0s, P * 24, st);
  cudaMallocAsync((void **)&b->d0obs, P * 16, st);
  cudaMallocAsync((void **)&b->iobs_s, P * 8, st);
  k_make_tiles<<<1, 1024, 0, st>>>(S, counts.as<unsigned int>(), tile_points, b->tile_start, b->tile_n,
                                   b->tile_slice, b->slice_tile0);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return bail(cuda_status(e, "k_make_tiles"));
  b->h_tstart.resize(b->T);
  b->h_tn.resize(b->T);
  cudaMemcpyAsync(b->h_tstart.data(), b->tile_start, b->T * 8, cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(b->h_tn.data(), b->tile_n, b->T * 4, cudaMemcpyDeviceToHost, st);
  cudaMallocAsync((void **)&b->tile_basis, b->T * 48, st);
  cudaMallocAsync((void **)&b->ab, P * 8, st);
  cudaMemsetAsync(flag.ptr, 0, 4, st);
  k_pack_tiles<128><<<(unsigned)b->T, 128, 0, st>>>(b->tile_start, b->tile_n, b->perm, x0, I_obs, b->x0s,
                                                  b->d0obs, b->iobs_s, b->tile_origin, b->tile_basis, b->ab,
                                                  flag.as<int>(), b->tile_radius);
  if (cudaError_t e = cudaGetLastError(); e != cudaSuccess) return bail(cuda_status(e, "k_pack_tiles"));
  int nonplanar = 0;
  cudaMemcpyAsync(&nonplanar, flag.ptr, 4, cudaMemcpyDeviceToHost, st);
  // host vectors must outlive the async copies
  if (cudaStreamSynchronize(st) != cudaSuccess) return bail(cuda_status(cudaGetLastError(), "pack"));
  b->planar = (nonplanar == 0);
  *out = b;
  return GSVR_OK;
}

int bin_prepare(gsvr_batch *b, int64_t K, int64_t N, cudaStream_t st, BinPlan *plan) {
  const int64_t PK = b->P * K;
  if ((int64_t)b->TP * K > 65535) return fail(GSVR_ERR_INVALID, "tile_points*K must be <= 65535");
  int bits = 1;
  while ((1ll << bits) < N) ++bits;
  plan->bits = bits;
  plan->fast = (int64_t)b->TP * K <= kBinCap && bits <= 31;
  // the per-tile path indexes pairs with 64-bit offsets; the device-wide
  // segmented sort of the fallback takes 32-bit item counts
  if (!plan->fast && PK > INT32_MAX) return fail(GSVR_ERR_INVALID, "P*K too large for one batch");
  int pbits = 1;
  while ((1 << pbits) <= b->TP) ++pbits;  // pixel ids < 2^pbits - 1 (pad key sorts last)
  plan->pbits = pbits;
  if (b->layout_K != K || !b->nl_off) {
    // padded per-tile segments: nbr_local 16-byte aligned (TMA bulk copies),
    // pair_pix chunk-transposed (C*256 slots per tile, coalesced per-lane reads);
    // totals on the host (allocation), offsets on the device
    int64_t a = 0, c = 0;
    for (int64_t t = 0; t < b->T; ++t) {
      const int64_t m = (int64_t)b->h_tn[t] * K;
      a += (nl_len(b->h_tn[t], (int)K) + 7) / 8 * 8;
      c += chunk_stride((int)m) * kChunkThreads;
    }
    if (b->nl_off) cudaFreeAsync(b->nl_off, st), b->nl_off = nullptr;
    if (b->pp_off) cudaFreeAsync(b->pp_off, st), b->pp_off = nullptr;
    if (b->nbr_local) cudaFreeAsync(b->nbr_local, st), b->nbr_local = nullptr;
    if (b->pair_pix) cudaFreeAsync(b->pair_pix, st), b->pair_pix = nullptr;
    GSVR_CUDA(cudaMallocAsync((void **)&b->nl_off, (b->T + 1) * 8, st));
    GSVR_CUDA(cudaMallocAsync((void **)&b->pp_off, (b->T + 1) * 8, st));
    GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_local, a * 2 + 64, st));
    GSVR_CUDA(cudaMallocAsync((void **)&b->pair_pix, c * 2 + 64, st));
    k_tile_layout<<<1, 1024, 0, st>>>(b->T, b->tile_n, K, b->nl_off, b->pp_off);
    GSVR_LAUNCH_CHECK("k_tile_layout");
    b->layout_K = K;
  }
  if (!b->uoff) GSVR_CUDA(cudaMallocAsync((void **)&b->uoff, (b->T + 1) * 4, st));
  GSVR_TRY(grow(b->ws[0], b->ws_cap[0], PK * 4, st));
  GSVR_TRY(grow(b->ws[1], b->ws_cap[1], PK * 2, st));
  GSVR_TRY(grow(b->ws[2], b->ws_cap[2], (b->T + 1) * 4, st));
  GSVR_CUDA(cudaMemsetAsync(b->ws[2], 0, (b->T + 1) * 4, st));
  GSVR_TRY(grow(b->rot_flag, b->cap_rot_flag, (size_t)b->T + 16, st));
  GSVR_CUDA(cudaMemsetAsync(b->rot_flag, 0, (size_t)b->T, st));
  if (plan->fast) {
    GSVR_TRY(ensure_smem((const void *)k_bin_sort, kBinSmem));
  }
  return GSVR_OK;
}

// Tiles [t0, t1) of the shared-memory path (plan.fast); nbr_int rows of those
// tiles must be in place.
// GSVR_BIN_SORT=1: always the sorting kernel (A/B; identical outputs)
static bool bin_hash_mode() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_BIN_SORT");
    return !(v && v[0] == '1');
  }();
  return on;
}

#ifdef GSVR_BIN_PROFILE
static void bin_profile_print(int64_t tiles, cudaStream_t st) {
  unsigned long long z[10];
  cudaMemcpyFromSymbolAsync(z, g_bin_phase, sizeof(z), 0, cudaMemcpyDeviceToHost, st);
  cudaStreamSynchronize(st);
  const double d = (double)tiles;
  std::fprintf(stderr, "BINPHASE tiles=%lld cycles/tile: init %.0f insert %.0f compact %.0f rank %.0f masks %.0f "
               "csr %.0f rotate %.0f transpose %.0f lists %.0f\n", (long long)tiles, z[0] / d, z[1] / d, z[2] / d,
               z[3] / d, z[4] / d, z[5] / d, z[6] / d, z[7] / d, z[8] / d);
  unsigned long long zero[10] = {0};
  cudaMemcpyToSymbolAsync(g_bin_phase, zero, sizeof(zero), 0, cudaMemcpyHostToDevice, st);
}
#else
static void bin_profile_print(int64_t, cudaStream_t) {}
#endif

int bin_sort_tiles(gsvr_batch *b, int64_t K, const BinPlan &plan, int64_t t0, int64_t t1, cudaStream_t st,
                   const int32_t *tile_list, BinSource ext) {
  if (t1 <= t0) return GSVR_OK;
  if (bin_hash_mode() && b->TP <= 256) {
    GSVR_TRY(ensure_smem((const void *)k_bin_hash, kHashSmem));
    if (plan.ov_list) {  // deferred: the caller flushes the overflow once
      k_bin_hash<<<(unsigned)(t1 - t0), kHashBlock, kHashSmem, st>>>(
          b->tile_start, b->tile_n, (int)K, b->nl_off, b->pp_off, b->nbr_int, b->nbr_local, b->pair_pix,
          (int32_t *)b->ws[0], (uint16_t *)b->ws[1], (int32_t *)b->ws[2], (int)t0, tile_list, ext, plan.ov_list,
          plan.ov_count, (int)pair_rotate_enabled());
      GSVR_LAUNCH_CHECK("k_bin_hash");
      bin_profile_print(t1 - t0, st);
      return GSVR_OK;
    }
    Scratch ov, nov;
    GSVR_TRY(ov.alloc((size_t)(t1 - t0) * 4, st));
    GSVR_TRY(nov.alloc(4, st));
    GSVR_CUDA(cudaMemsetAsync(nov.ptr, 0, 4, st));
    k_bin_hash<<<(unsigned)(t1 - t0), kHashBlock, kHashSmem, st>>>(
        b->tile_start, b->tile_n, (int)K, b->nl_off, b->pp_off, b->nbr_int, b->nbr_local, b->pair_pix,
        (int32_t *)b->ws[0], (uint16_t *)b->ws[1], (int32_t *)b->ws[2], (int)t0, tile_list, ext,
        ov.as<int32_t>(), nov.as<int>(), (int)pair_rotate_enabled());
    GSVR_LAUNCH_CHECK("k_bin_hash");
    bin_profile_print(t1 - t0, st);
    int n_ov = 0;
    GSVR_CUDA(cudaMemcpyAsync(&n_ov, nov.ptr, 4, cudaMemcpyDeviceToHost, st));
    GSVR_CUDA(cudaStreamSynchronize(st));
    if (n_ov == 0) return GSVR_OK;
    k_bin_sort<<<(unsigned)n_ov, kBinBlock, kBinSmem, st>>>(
        b->tile_start, b->tile_n, (int)K, plan.bits, plan.pbits, b->nl_off, b->pp_off, b->nbr_int, b->nbr_local,
        b->pair_pix, (int32_t *)b->ws[0], (uint16_t *)b->ws[1], (int32_t *)b->ws[2], 0, ov.as<int32_t>(), ext,
        b->rot_flag);
    GSVR_LAUNCH_CHECK("k_bin_sort (overflow tiles)");
    return GSVR_OK;
  }
  k_bin_sort<<<(unsigned)(t1 - t0), kBinBlock, kBinSmem, st>>>(
      b->tile_start, b->tile_n, (int)K, plan.bits, plan.pbits, b->nl_off, b->pp_off, b->nbr_int, b->nbr_local,
      b->pair_pix, (int32_t *)b->ws[0], (uint16_t *)b->ws[1], (int32_t *)b->ws[2], (int)t0, tile_list, ext,
      b->rot_flag);
  GSVR_LAUNCH_CHECK("k_bin_sort");
  return GSVR_OK;
}

int bin_flush_overflow(gsvr_batch *b, int64_t K, const BinPlan &plan, cudaStream_t st, BinSource ext) {
  if (!plan.ov_list) return GSVR_OK;
  int n_ov = 0;
  GSVR_CUDA(cudaMemcpyAsync(&n_ov, plan.ov_count, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  if (n_ov == 0) return GSVR_OK;
  k_bin_sort<<<(unsigned)n_ov, kBinBlock, kBinSmem, st>>>(
      b->tile_start, b->tile_n, (int)K, plan.bits, plan.pbits, b->nl_off, b->pp_off, b->nbr_int, b->nbr_local,
      b->pair_pix, (int32_t *)b->ws[0], (uint16_t *)b->ws[1], (int32_t *)b->ws[2], 0, plan.ov_list, ext,
      b->rot_flag);
  GSVR_LAUNCH_CHECK("k_bin_sort (overflow tiles)");
  return GSVR_OK;
}

// Large tiles: device-wide segmented radix sort, then one pass per tile.
static int bin_sort_fallback(gsvr_batch *b, int64_t K, const BinPlan &plan, cudaStream_t st) {
  const int64_t PK = b->P * K;
  const int bits = plan.bits;
  int32_t *gid_tmp = (int32_t *)b->ws[0], *nuniq = (int32_t *)b->ws[2];
  uint16_t *csr_tmp = (uint16_t *)b->ws[1];
  Scratch vals, skeys, svals, off, tmp;
  GSVR_TRY(vals.alloc(PK * 4, st));
  GSVR_TRY(skeys.alloc(PK * 4, st));
  GSVR_TRY(svals.alloc(PK * 4, st));
  GSVR_TRY(off.alloc((b->T + 1) * 8, st));
  k_pair_positions<<<(unsigned)b->T, 256, 0, st>>>(b->tile_start, b->tile_n, K, vals.as<int32_t>());
  k_segment_offsets<<<grid_for(b->T, 256), 256, 0, st>>>(b->T, b->tile_start, b->tile_n, K, off.as<int64_t>());
  size_t tbytes = 0;
  const int64_t *ob = off.as<int64_t>();
  cub::DeviceSegmentedRadixSort::SortPairs(nullptr, tbytes, b->nbr_int, skeys.as<int32_t>(), vals.as<int32_t>(),
                                           svals.as<int32_t>(), (int)PK, (int)b->T, ob, ob + 1, 0, bits, st);
  GSVR_TRY(tmp.alloc(tbytes, st));
  cub::DeviceSegmentedRadixSort::SortPairs(tmp.ptr, tbytes, b->nbr_int, skeys.as<int32_t>(), vals.as<int32_t>(),
                                           svals.as<int32_t>(), (int)PK, (int)b->T, ob, ob + 1, 0, bits, st);
  GSVR_LAUNCH_CHECK("segmented sort");
  k_bin_tiles<256><<<(unsigned)b->T, 256, 0, st>>>(b->tile_start, b->tile_n, K, skeys.as<int32_t>(),
                                                   svals.as<int32_t>(), b->nl_off, b->pp_off,
                                                   b->nbr_local, b->pair_pix, gid_tmp, csr_tmp, nuniq,
                                                   b->rot_flag);
  GSVR_LAUNCH_CHECK("k_bin_tiles");
  return GSVR_OK;
}

// Per-tile unique counts -> offsets, compacted (gid, csr), inverse record map.

int bin_finish(gsvr_batch *b, int64_t K, int64_t N, const BinPlan &plan, cudaStream_t st) {
  StageTrace tr("bin", st);
  const int bits = plan.bits;
  int32_t *gid_tmp = (int32_t *)b->ws[0], *nuniq = (int32_t *)b->ws[2];
  uint16_t *csr_tmp = (uint16_t *)b->ws[1];
  size_t sbytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, sbytes, nuniq, b->uoff, (int)(b->T + 1), st);
  GSVR_TRY(grow(b->ws[3], b->ws_cap[3], sbytes, st));
  cub::DeviceScan::ExclusiveSum(b->ws[3], sbytes, nuniq, b->uoff, (int)(b->T + 1), st);
  int32_t U = 0;
  GSVR_CUDA(cudaMemcpyAsync(&U, b->uoff + b->T, 4, cudaMemcpyDeviceToHost, st));
  // max unique per tile (decides whether the overflow record buffer is needed)
  std::vector<int32_t> hu(b->T + 1);
  GSVR_CUDA(cudaMemcpyAsync(hu.data(), b->uoff, (b->T + 1) * 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  int mx = 0;
  b->h_nu.resize(b->T);
  for (int64_t t = 0; t < b->T; ++t) {
    b->h_nu[t] = hu[t + 1] - hu[t];
    mx = std::max(mx, b->h_nu[t]);
  }
  b->buckets_valid = false;
  GSVR_TRY(grow(b->gid, b->cap_gid, (size_t)U * 4 + 16, st));
  GSVR_TRY(grow(b->csr, b->cap_csr, ((size_t)U + b->T) * 2 + 16, st));
  // global record pages are read only by tiles whose unique-Gaussian list
  // exceeds a kernel's shared-memory page (never at cfg1-4): allocated only
  // then (U x 80 bytes: 3.5 GB at cfg3 otherwise)
  if (mx > kMinRecordPage) {
    GSVR_TRY(grow(b->rec, b->cap_rec, (size_t)U * 80 + 16, st));
  } else if (b->rec) {
    cudaFreeAsync(b->rec, st);
    b->rec = nullptr;
    b->cap_rec = 0;
  }
  k_compact_unique<<<(unsigned)b->T, 256, 0, st>>>(b->tile_start, b->tile_n, K, b->uoff, gid_tmp, csr_tmp,
                                                   b->gid, b->csr);
  GSVR_LAUNCH_CHECK("k_compact_unique");
  if (pair_rotate_enabled() && b->TP <= 256) {
    k_pair_rotate<<<(unsigned)b->T, 256, 0, st>>>(b->tile_n, (int)K, b->uoff, b->csr, b->pp_off, b->rot_flag,
                                                  b->pair_pix);
    GSVR_LAUNCH_CHECK("k_pair_rotate");
  }
  tr.mark("compact");
  // inverse map Gaussian -> its (tile, Gaussian) records, tile order (stable radix sort)
  GSVR_TRY(grow(b->jr_idx, b->cap_jr_idx, (size_t)U * 4 + 16, st));
  GSVR_TRY(grow(b->jr_ptr, b->cap_jr_ptr, (size_t)(N + 1) * 4, st));
  GSVR_TRY(grow(b->gpart, b->cap_gpart, (size_t)U * 40 + 16, st));
  {
    GSVR_TRY(grow(b->ws[4], b->ws_cap[4], (size_t)U * 4 + 16, st));
    GSVR_TRY(grow(b->ws[5], b->ws_cap[5], (size_t)U * 4 + 16, st));
    int32_t *iota = (int32_t *)b->ws[4], *skey = (int32_t *)b->ws[5];
    k_iota<<<grid_for(U, 256), 256, 0, st>>>(U, iota);
    size_t tb = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb, b->gid, skey, iota, b->jr_idx, (int)U, 0, bits, st);
    GSVR_TRY(grow(b->ws[3], b->ws_cap[3], tb, st));
    cub::DeviceRadixSort::SortPairs(b->ws[3], tb, b->gid, skey, iota, b->jr_idx, (int)U, 0, bits, st);
    k_lower_bounds<<<grid_for(N + 1, 256), 256, 0, st>>>(N, U, skey, b->jr_ptr);
    GSVR_LAUNCH_CHECK("inverse record map");
    // gather order: Gaussians sorted by the position of their first record, so
    // a warp's Gaussians read neighbouring (tile-major) partials
    Scratch fk, fk2, fv, ftmp;
    GSVR_TRY(fk.alloc((size_t)N * 4, st));
    GSVR_TRY(fk2.alloc((size_t)N * 4, st));
    GSVR_TRY(fv.alloc((size_t)N * 4, st));
    GSVR_TRY(grow(b->gorder, b->cap_gorder, (size_t)N * 4 + 16, st));
    k_first_record<<<grid_for(N, 256), 256, 0, st>>>(N, b->jr_ptr, b->jr_idx, fk.as<uint32_t>(), fv.as<int32_t>());
    int kbits = 1;
    while ((1ll << kbits) <= U) ++kbits;
    size_t tb2 = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, tb2, fk.as<uint32_t>(), fk2.as<uint32_t>(), fv.as<int32_t>(),
                                    b->gorder, (int)N, 0, kbits, st);
    GSVR_TRY(ftmp.alloc(tb2, st));
    cub::DeviceRadixSort::SortPairs(ftmp.ptr, tb2, fk.as<uint32_t>(), fk2.as<uint32_t>(), fv.as<int32_t>(),
                                    b->gorder, (int)N, 0, kbits, st);
    GSVR_LAUNCH_CHECK("gather order");
  }
  tr.mark("inverse");
  b->K = K;
  b->N = N;
  b->U = U;
  b->max_unique = mx;
  return GSVR_OK;
}

int gather_nbr_rows(gsvr_batch *b, int64_t K, int64_t N, const void *nbr, int nbr_i64, int64_t i0, int64_t i1,
                    int *bad, cudaStream_t st) {
  if (i1 <= i0) return GSVR_OK;
  const unsigned grid = grid_for((i1 - i0) * 32, 256);
  if (nbr_i64)
    k_gather_nbr<int64_t><<<grid, 256, 0, st>>>(i0, i1, (int)K, N, b->perm, (const int64_t *)nbr, b->nbr_int, bad);
  else
    k_gather_nbr<int32_t><<<grid, 256, 0, st>>>(i0, i1, (int)K, N, b->perm, (const int32_t *)nbr, b->nbr_int, bad);
  GSVR_LAUNCH_CHECK("k_gather_nbr");
  return GSVR_OK;
}

int batch_bin_internal(gsvr_batch *b, int64_t K, int64_t N, cudaStream_t st) {
  StageTrace tr("bin", st);
  BinPlan plan;
  GSVR_TRY(bin_prepare(b, K, N, st, &plan));
  tr.mark("alloc");
  if (plan.fast) {
    GSVR_TRY(bin_sort_tiles(b, K, plan, 0, b->T, st));
  } else {
    GSVR_TRY(bin_sort_fallback(b, K, plan, st));
  }
  tr.mark("sort");
  return bin_finish(b, K, N, plan, st);
}

}  // namespace gsvr

void gsvr_batch::release_binning() {
  cudaStream_t st = owner_stream;
  if (nbr_next) cudaFreeAsync(nbr_next, st), nbr_next = nullptr;
  seeds_valid = false;
  for (void *p : {(void *)nbr_int, (void *)nbr_local, (void *)pair_pix, (void *)nl_off, (void *)pp_off,
                  (void *)uoff, (void *)gid, (void *)gpart, (void *)jr_ptr, (void *)jr_idx, (void *)gorder,
                  (void *)csr, (void *)rec, (void *)rot_flag})
    if (p) cudaFreeAsync(p, st);
  nbr_int = nullptr, nbr_local = nullptr, pair_pix = nullptr, uoff = nullptr, gid = nullptr;
  nl_off = nullptr, pp_off = nullptr, gpart = nullptr, jr_ptr = nullptr, jr_idx = nullptr, gorder = nullptr;
  csr = nullptr, rec = nullptr, rot_flag = nullptr, cap_rot_flag = 0;
  for (int i = 0; i < 6; ++i) {
    if (ws[i]) cudaFreeAsync(ws[i], st);
    ws[i] = nullptr, ws_cap[i] = 0;
  }
  cap_gid = cap_csr = cap_rec = cap_gpart = cap_jr_idx = cap_jr_ptr = cap_gorder = 0;
  layout_K = 0;
  K = N = U = 0;
}

gsvr_batch::~gsvr_batch() {
  release_binning();
  cudaStream_t st = owner_stream;
  if (ws_disp) cudaFreeAsync(ws_disp, st);
  if (ws_grec) cudaFreeAsync(ws_grec, st);
  if (ws_brec) cudaFreeAsync(ws_brec, st);
  if (ws_knn_scr) cudaFreeAsync(ws_knn_scr, st);
  if (ws_knn_fb) cudaFreeAsync(ws_knn_fb, st);
  if (gpos) cudaFreeAsync(gpos, st);
  if (tile_buckets) cudaFreeAsync(tile_buckets, st);
  for (void *p : {(void *)perm, (void *)sid_s, (void *)x0s, (void *)d0obs, (void *)iobs_s, (void *)tile_start,
                  (void *)tile_n, (void *)tile_slice, (void *)tile_origin, (void *)tile_radius, (void *)tile_basis, (void *)ab, (void *)tpart, (void *)slice_tile0})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
}

using namespace gsvr;

extern "C" {

int gsvr_batch_create(int64_t P, int64_t S, const double *x0pts, const int32_t *sid, const double *I_obs,
                      int tile_points, gsvr_batch **out, void *stream) {
  return batch_create(P, S, x0pts, sid, I_obs, tile_points, out, as_stream(stream));
}

void gsvr_batch_free(gsvr_batch *batch) { delete batch; }
int64_t gsvr_batch_tiles(const gsvr_batch *b) { return b ? b->T : 0; }
const int32_t *gsvr_batch_perm(const gsvr_batch *b) { return b ? b->perm : nullptr; }
int64_t gsvr_batch_tile_gaussians(const gsvr_batch *b) { return b ? b->U : 0; }

int gsvr_batch_set_observed(gsvr_batch *b, const double *I_obs, void *stream) {
  cudaStream_t st = as_stream(stream);
  k_set_observed<<<grid_for(b->P, 256), 256, 0, st>>>(b->P, b->perm, I_obs, b->d0obs, b->iobs_s);
  GSVR_LAUNCH_CHECK("k_set_observed");
  return GSVR_OK;
}

int gsvr_batch_bin(gsvr_batch *b, int64_t K, int64_t N, const void *nbr, int nbr_i64, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (K < 1 || N < 1) return fail(GSVR_ERR_INVALID, "K and N must be positive");
  if (b->nbr_int && b->K != K) b->release_binning();
  if (!b->nbr_int) GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_int, b->P * K * 4, st));
  b->seeds_valid = false;  // caller lists may repeat ids: never a pruning bound
  b->gpos_N = 0;           // no index: rows stay in id order
  Scratch flag;
  GSVR_TRY(flag.alloc(4, st));
  GSVR_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, st));
  if (nbr_i64)
    k_gather_nbr<int64_t><<<grid_for(b->P * 32, 256), 256, 0, st>>>(0, b->P, (int)K, N, b->perm,
                                                                    (const int64_t *)nbr, b->nbr_int, flag.as<int>());
  else
    k_gather_nbr<int32_t><<<grid_for(b->P * 32, 256), 256, 0, st>>>(0, b->P, (int)K, N, b->perm,
                                                                    (const int32_t *)nbr, b->nbr_int, flag.as<int>());
  GSVR_LAUNCH_CHECK("k_gather_nbr");
  int bad = 0;
  GSVR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(GSVR_ERR_INVALID, "neighbor id out of range");
  return batch_bin_internal(b, K, N, st);
}

int gsvr_batch_neighbors(const gsvr_batch *b, int64_t *out, void *stream) {
  if (!b->nbr_int) return fail(GSVR_ERR_INVALID, "batch has no neighbour lists");
  cudaStream_t st = as_stream(stream);
  k_scatter_nbr<<<grid_for(b->P * b->K, 256), 256, 0, st>>>(b->P, b->K, b->perm, b->nbr_int, out);
  GSVR_LAUNCH_CHECK("k_scatter_nbr");
  return GSVR_OK;
}

int gsvr_batch_tile_info(const gsvr_batch *b, int64_t *tile_start, int32_t *tile_n, int32_t *tile_slice,
                         int32_t *uoff, int32_t *gid, int32_t *perm, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (perm) GSVR_CUDA(cudaMemcpyAsync(perm, b->perm, b->P * 4, cudaMemcpyDeviceToDevice, st));
  if (tile_start) GSVR_CUDA(cudaMemcpyAsync(tile_start, b->tile_start, b->T * 8, cudaMemcpyDeviceToDevice, st));
  if (tile_n) GSVR_CUDA(cudaMemcpyAsync(tile_n, b->tile_n, b->T * 4, cudaMemcpyDeviceToDevice, st));
  if (tile_slice) GSVR_CUDA(cudaMemcpyAsync(tile_slice, b->tile_slice, b->T * 4, cudaMemcpyDeviceToDevice, st));
  if (uoff || gid) {
    if (!b->uoff) return fail(GSVR_ERR_INVALID, "batch has no binning");
    if (uoff) GSVR_CUDA(cudaMemcpyAsync(uoff, b->uoff, (b->T + 1) * 4, cudaMemcpyDeviceToDevice, st));
    if (gid) GSVR_CUDA(cudaMemcpyAsync(gid, b->gid, b->U * 4, cudaMemcpyDeviceToDevice, st));
  }
  return GSVR_OK;
}

int gsvr_batch_tile_geometry(const gsvr_batch *b, double *origin, double *basis, float *ab, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (origin) GSVR_CUDA(cudaMemcpyAsync(origin, b->tile_origin, b->T * 24, cudaMemcpyDeviceToDevice, st));
  if (basis) GSVR_CUDA(cudaMemcpyAsync(basis, b->tile_basis, b->T * 48, cudaMemcpyDeviceToDevice, st));
  if (ab) GSVR_CUDA(cudaMemcpyAsync(ab, b->ab, b->P * 8, cudaMemcpyDeviceToDevice, st));
  return GSVR_OK;
}

}  // extern "C"
