// simulate.cu -- acquisition simulator's PSF quadrature (simulate.py:142-205).
//
// gsvr_psf_quadrature: for every pixel centre p, the Gaussian-weighted tensor
// quadrature of a ground-truth raster over slice-frame offsets (a, b, c) along
// that pixel's slice axes, each sample trilinearly interpolated (zero outside
// the raster).  Data generation for the fetal-scale configs (SURVEY.md §8f row
// 4), not part of the per-epoch path.
//
// The reference evaluates this in float64 without FMA contraction (numba,
// fastmath off); every product and sum below is an explicitly rounded
// __dmul_rn / __dadd_rn / __dsub_rn in the reference's order, so results agree
// with it to the last bits.  One thread per pixel; the node tables live in
// shared memory; neighbouring threads (neighbouring pixels) read overlapping
// raster neighbourhoods, which L1/L2 serve.
#include "common.cuh"

namespace gsvr {

constexpr int kMaxQuadNodes = 128;

__device__ __forceinline__ double dm(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double da(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double ds(double a, double b) { return __dsub_rn(a, b); }

// simulate.py:142-165 (x-major raster, vol[(x * ny + y) * nz + z])
__device__ inline double trilinear(const double *__restrict__ vol, int nx, int ny, int nz, double ix, double iy,
                                   double iz) {
  if (ix < 0.0 || iy < 0.0 || iz < 0.0 || ix > (double)(nx - 1) || iy > (double)(ny - 1) || iz > (double)(nz - 1))
    return 0.0;
  int x0 = (int)ix, y0 = (int)iy, z0 = (int)iz;
  if (x0 > nx - 2) x0 = nx - 2;
  if (y0 > ny - 2) y0 = ny - 2;
  if (z0 > nz - 2) z0 = nz - 2;
  const double fx = ds(ix, (double)x0), fy = ds(iy, (double)y0), fz = ds(iz, (double)z0);
  const double gx = ds(1.0, fx), gy = ds(1.0, fy), gz = ds(1.0, fz);
  auto V = [&](int x, int y, int z) { return __ldg(vol + ((int64_t)x * ny + y) * nz + z); };
  const double c00 = da(dm(V(x0, y0, z0), gx), dm(V(x0 + 1, y0, z0), fx));
  const double c10 = da(dm(V(x0, y0 + 1, z0), gx), dm(V(x0 + 1, y0 + 1, z0), fx));
  const double c01 = da(dm(V(x0, y0, z0 + 1), gx), dm(V(x0 + 1, y0, z0 + 1), fx));
  const double c11 = da(dm(V(x0, y0 + 1, z0 + 1), gx), dm(V(x0 + 1, y0 + 1, z0 + 1), fx));
  const double c0 = da(dm(c00, gy), dm(c10, fy));
  const double c1 = da(dm(c01, gy), dm(c11, fy));
  return da(dm(c0, gz), dm(c1, fz));
}

struct QuadArgs {
  const double *vol;
  int nx, ny, nz;
  double inv[12];  // inverse affine rows 0..2 (x, y, z, 1)
  int64_t M;
  const double *centers;  // (M, 3)
  const int32_t *sid;     // (M,) slice of each centre, or null (axes[0] for all)
  const double *axes;     // (S, 3, 3) row-major: column k = k-th slice axis in world
  const double *nodes;    // [offx wx | offy wy | offz wz]
  int n0, n1, n2;
  double *out;
};

// simulate.py:168-205
__global__ void __launch_bounds__(128) k_psf_quadrature(QuadArgs q) {
  __shared__ double sn[6 * kMaxQuadNodes];
  const int ntot = 2 * (q.n0 + q.n1 + q.n2);
  for (int i = threadIdx.x; i < ntot; i += blockDim.x) sn[i] = q.nodes[i];
  __syncthreads();
  const double *offx = sn, *wx = offx + q.n0, *offy = wx + q.n0, *wy = offy + q.n1, *offz = wy + q.n1,
               *wz = offz + q.n2;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < q.M; p += (int64_t)gridDim.x * blockDim.x) {
    const double *A = q.axes + 9 * (q.sid ? (int64_t)q.sid[p] : 0);
    const double cx = q.centers[3 * p], cy = q.centers[3 * p + 1], cz = q.centers[3 * p + 2];
    double acc = 0.0;
    for (int ia = 0; ia < q.n0; ++ia) {
      const double a = offx[ia];
      const double qx = da(cx, dm(A[0], a)), qy = da(cy, dm(A[3], a)), qz = da(cz, dm(A[6], a));
      for (int ib = 0; ib < q.n1; ++ib) {
        const double b = offy[ib];
        const double rx = da(qx, dm(A[1], b)), ry = da(qy, dm(A[4], b)), rz = da(qz, dm(A[7], b));
        const double wab = dm(wx[ia], wy[ib]);
        for (int ic = 0; ic < q.n2; ++ic) {
          const double c = offz[ic];
          const double px = da(rx, dm(A[2], c)), py = da(ry, dm(A[5], c)), pz = da(rz, dm(A[8], c));
          const double ix = da(da(da(dm(q.inv[0], px), dm(q.inv[1], py)), dm(q.inv[2], pz)), q.inv[3]);
          const double iy = da(da(da(dm(q.inv[4], px), dm(q.inv[5], py)), dm(q.inv[6], pz)), q.inv[7]);
          const double iz = da(da(da(dm(q.inv[8], px), dm(q.inv[9], py)), dm(q.inv[10], pz)), q.inv[11]);
          acc = da(acc, dm(dm(wab, wz[ic]), trilinear(q.vol, q.nx, q.ny, q.nz, ix, iy, iz)));
        }
      }
    }
    q.out[p] = acc;
  }
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_psf_quadrature(int64_t nx, int64_t ny, int64_t nz, const double *vol, const double *inv_affine, int64_t M,
                        const double *centers, const int32_t *sid, const double *axes, int64_t n0, int64_t n1,
                        int64_t n2, const double *nodes, double *out, void *stream) {
  if (M == 0) return GSVR_OK;
  if (nx < 2 || ny < 2 || nz < 2) return fail(GSVR_ERR_INVALID, "raster must be at least 2x2x2");
  if (nx * ny * nz > (int64_t)1 << 40) return fail(GSVR_ERR_INVALID, "raster too large");
  if (n0 < 1 || n1 < 1 || n2 < 1 || n0 > kMaxQuadNodes || n1 > kMaxQuadNodes || n2 > kMaxQuadNodes)
    return fail(GSVR_ERR_INVALID, "quadrature nodes per axis must be in [1, %d]", kMaxQuadNodes);
  if (!vol || !inv_affine || !centers || !axes || !nodes || !out)
    return fail(GSVR_ERR_INVALID, "null array");
  cudaStream_t st = as_stream(stream);
  QuadArgs q;
  q.vol = vol;
  q.nx = (int)nx;
  q.ny = (int)ny;
  q.nz = (int)nz;
  for (int i = 0; i < 12; ++i) q.inv[i] = inv_affine[i];  // host array (3x4)
  q.M = M;
  q.centers = centers;
  q.sid = sid;
  q.axes = axes;
  q.nodes = nodes;
  q.n0 = (int)n0;
  q.n1 = (int)n1;
  q.n2 = (int)n2;
  q.out = out;
  k_psf_quadrature<<<grid_for(M, 128, 148 * 64), 128, 0, st>>>(q);
  GSVR_LAUNCH_CHECK("k_psf_quadrature");
  return GSVR_OK;
}

}  // extern "C"
