/*
 * gsvr_oracle.c -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
 *
 * This file is the parity checker, not the product.  Only tests/, the
 * __graft_entry__.smoke() check and bench.py's cpu_baseline / --impl reference
 * legs may load it.  The product path (paper_2512_11624_b200/) never links it.
 *
 * It restates, in plain C + OpenMP and in float64 like the reference, the
 * numba kernels of /root/reference/pkg/src/gsvr/kernels.py:
 *
 *   oracle_render_forward       <- kernels.py:41-75   (clamp-at-EXP_CLAMP forward)
 *   oracle_train_step_backward  <- kernels.py:78-198  (drop-below-EXP_CLAMP fused
 *                                   forward + L1 + analytic gradients, fixed
 *                                   block partition, per-block private buffers)
 *   oracle_default_block_count  <- kernels.py:201-203
 *   oracle_knn_query            <- knn.py:43-75 (exact top-K with the reference's
 *                                   tie rules; brute force, see below)
 *
 * Parity pin: tests/test_oracle_golden.py checks every function here against
 * golden vectors produced by the reference itself (oracle/gen_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define EXP_CLAMP (-80.0) /* kernels.py:25 */

/* kernels.py:28-38: cofactor inverse of a packed symmetric 3x3. */
static inline void inv_sym3(double a00, double a01, double a02, double a11,
                            double a12, double a22, double *m) {
  double c00 = a11 * a22 - a12 * a12;
  double c01 = a02 * a12 - a01 * a22;
  double c02 = a01 * a12 - a02 * a11;
  double c11 = a00 * a22 - a02 * a02;
  double c12 = a01 * a02 - a00 * a12;
  double c22 = a00 * a11 - a01 * a01;
  double det = a00 * c00 + a01 * c01 + a02 * c02;
  double idet = 1.0 / det;
  m[0] = c00 * idet; m[1] = c01 * idet; m[2] = c02 * idet;
  m[3] = c11 * idet; m[4] = c12 * idet; m[5] = c22 * idet;
}

/* Thread count of the parallel loops (timing harness: all host threads even
 * when a launcher exported OMP_NUM_THREADS=1).  Returns the count in effect. */
int oracle_set_threads(int n) {
#ifdef _OPENMP
  if (n > 0) omp_set_num_threads(n);
  return omp_get_max_threads();
#else
  (void)n;
  return 1;
#endif
}

int oracle_default_block_count(int64_t n_points) {
  /* kernels.py:201-203 */
  if (n_points < 1) return 1;
  return n_points < 16 ? (int)n_points : 16;
}

/* kernels.py:41-75.  points (M,3), psf6 (M,6), sigma (M,), nbr (M,K) int64,
 * mu (N,3), cov6 (N,6), cvals (N,) -> out (M,). */
void oracle_render_forward(int64_t M, int64_t K, const double *points,
                           const double *psf6, const double *sigma,
                           const int64_t *nbr, const double *mu,
                           const double *cov6, const double *cvals,
                           double delta, double *out) {
#pragma omp parallel for schedule(static)
  for (int64_t p = 0; p < M; ++p) {
    const double x0 = points[3 * p], x1 = points[3 * p + 1], x2 = points[3 * p + 2];
    const double *ps = psf6 + 6 * p;
    double num = 0.0, den = delta;
    for (int64_t k = 0; k < K; ++k) {
      const int64_t j = nbr[p * K + k];
      const double *c = cov6 + 6 * j;
      double m[6];
      inv_sym3(c[0] + ps[0], c[1] + ps[1], c[2] + ps[2], c[3] + ps[3],
               c[4] + ps[4], c[5] + ps[5], m);
      double v0 = x0 - mu[3 * j], v1 = x1 - mu[3 * j + 1], v2 = x2 - mu[3 * j + 2];
      double w0 = m[0] * v0 + m[1] * v1 + m[2] * v2;
      double w1 = m[1] * v0 + m[3] * v1 + m[4] * v2;
      double w2 = m[2] * v0 + m[4] * v1 + m[5] * v2;
      double u = -0.5 * (v0 * w0 + v1 * w1 + v2 * w2);
      if (u < EXP_CLAMP) u = EXP_CLAMP;
      double e = exp(u);
      num += cvals[j] * e;
      den += e;
    }
    out[p] = sigma[p] * num / den;
  }
}

/* kernels.py:78-198.  Gradient buffers carry a leading block axis of size
 * n_blocks and must be zero-filled by the caller (train.py:247-253). */
void oracle_train_step_backward(
    int64_t P, int64_t K, int64_t S, int64_t N, const double *x0pts,
    const int32_t *sid, const double *Rc, const double *tvec,
    const double *psf6s, const double *sigma_s, const double *wdata_s,
    const double *I_obs, const int64_t *nbr, const double *mu,
    const double *cov6, const double *cvals, double delta, int n_blocks,
    double *I_hat, double *absres, double *dmu, double *dcov6, double *dc,
    double *dt, double *dRc, double *dpsf6, double *dsigraw) {
#pragma omp parallel for schedule(dynamic, 1)
  for (int b = 0; b < n_blocks; ++b) {
    const int64_t lo = (int64_t)b * P / n_blocks;
    const int64_t hi = (int64_t)(b + 1) * P / n_blocks;
    double *e_buf = (double *)malloc(sizeof(double) * (size_t)(K > 0 ? K : 1));
    double *w_buf = (double *)malloc(sizeof(double) * 3 * (size_t)(K > 0 ? K : 1));
    double *bmu = dmu + (size_t)b * N * 3, *bcov = dcov6 + (size_t)b * N * 6;
    double *bc = dc + (size_t)b * N, *bt = dt + (size_t)b * S * 3;
    double *bR = dRc + (size_t)b * S * 9, *bp = dpsf6 + (size_t)b * S * 6;
    double *bs = dsigraw + (size_t)b * S;
    for (int64_t p = lo; p < hi; ++p) {
      const int s = sid[p];
      const double *R = Rc + 9 * s;
      const double a0 = x0pts[3 * p], a1 = x0pts[3 * p + 1], a2 = x0pts[3 * p + 2];
      const double x0 = R[0] * a0 + R[1] * a1 + R[2] * a2 + tvec[3 * s];
      const double x1 = R[3] * a0 + R[4] * a1 + R[5] * a2 + tvec[3 * s + 1];
      const double x2 = R[6] * a0 + R[7] * a1 + R[8] * a2 + tvec[3 * s + 2];
      const double *ps = psf6s + 6 * s;
      double num = 0.0, den = delta;
      for (int64_t k = 0; k < K; ++k) {
        const int64_t j = nbr[p * K + k];
        const double *c = cov6 + 6 * j;
        double m[6];
        inv_sym3(c[0] + ps[0], c[1] + ps[1], c[2] + ps[2], c[3] + ps[3],
                 c[4] + ps[4], c[5] + ps[5], m);
        double v0 = x0 - mu[3 * j], v1 = x1 - mu[3 * j + 1], v2 = x2 - mu[3 * j + 2];
        double w0 = m[0] * v0 + m[1] * v1 + m[2] * v2;
        double w1 = m[1] * v0 + m[3] * v1 + m[4] * v2;
        double w2 = m[2] * v0 + m[4] * v1 + m[5] * v2;
        double u = -0.5 * (v0 * w0 + v1 * w1 + v2 * w2);
        double e = (u < EXP_CLAMP) ? 0.0 : exp(u); /* drop, kernels.py:123-126 */
        e_buf[k] = e;
        w_buf[3 * k] = w0; w_buf[3 * k + 1] = w1; w_buf[3 * k + 2] = w2;
        num += cvals[j] * e;
        den += e;
      }
      const double ratio = num / den;
      const double ihat = sigma_s[s] * ratio;
      I_hat[p] = ihat;
      const double r = ihat - I_obs[p];
      absres[p] = fabs(r);
      double g = (r > 0.0) ? wdata_s[s] : ((r < 0.0) ? -wdata_s[s] : 0.0);
      bs[s] += g * ratio;
      const double gout = g * sigma_s[s];
      const double gnum = gout / den;
      const double gden = -gout * ratio / den;
      double gx0 = 0.0, gx1 = 0.0, gx2 = 0.0;
      for (int64_t k = 0; k < K; ++k) {
        const double e = e_buf[k];
        if (e == 0.0) continue;
        const int64_t j = nbr[p * K + k];
        bc[j] += gnum * e;
        const double a = (gnum * cvals[j] + gden) * e;
        const double w0 = w_buf[3 * k], w1 = w_buf[3 * k + 1], w2 = w_buf[3 * k + 2];
        bmu[3 * j] += a * w0; bmu[3 * j + 1] += a * w1; bmu[3 * j + 2] += a * w2;
        gx0 -= a * w0; gx1 -= a * w1; gx2 -= a * w2;
        const double ha = 0.5 * a;
        const double s00 = ha * w0 * w0, s01 = ha * w0 * w1, s02 = ha * w0 * w2;
        const double s11 = ha * w1 * w1, s12 = ha * w1 * w2, s22 = ha * w2 * w2;
        double *gc = bcov + 6 * j;
        gc[0] += s00; gc[1] += s01; gc[2] += s02; gc[3] += s11; gc[4] += s12; gc[5] += s22;
        double *gp = bp + 6 * s;
        gp[0] += s00; gp[1] += s01; gp[2] += s02; gp[3] += s11; gp[4] += s12; gp[5] += s22;
      }
      bt[3 * s] += gx0; bt[3 * s + 1] += gx1; bt[3 * s + 2] += gx2;
      double *gR = bR + 9 * s;
      gR[0] += gx0 * a0; gR[1] += gx0 * a1; gR[2] += gx0 * a2;
      gR[3] += gx1 * a0; gR[4] += gx1 * a1; gR[5] += gx1 * a2;
      gR[6] += gx2 * a0; gR[7] += gx2 * a1; gR[8] += gx2 * a2;
    }
    free(e_buf);
    free(w_buf);
  }
}

/* ------------------------------------------------------------------------ */
/* knn.py:43-75 restated by brute force.
 *
 * The reference asks cKDTree for k_eff = min(K+1, N) neighbours.  cKDTree's
 * distance is sqrt(((dx*dx + dy*dy) + dz*dz)) in float64 (checked bit-exact
 * against scipy 1.18 in oracle/gen_golden.py).  Rows come back ordered by
 * (distance, index) (knn.py:58-65; with no ties anywhere the distance order is
 * already strict).  A row whose distances at positions K-1 and K are equal is
 * re-resolved by brute force ordered by (d2, index) (knn.py:67-74).
 * Both orders are restated here; d2 is the unrounded square sum, so the two
 * differ only where sqrt() maps distinct d2 to one distance. */
typedef struct {
  double d2;
  int64_t idx;
} cand_t;

static inline int cand_less(const cand_t *a, const cand_t *b) {
  return (a->d2 < b->d2) || (a->d2 == b->d2 && a->idx < b->idx);
}

static inline double sq_dist(const double *m, const double *p) {
  double dx = m[0] - p[0], dy = m[1] - p[1], dz = m[2] - p[2];
  double s = dx * dx;
  s = s + dy * dy;
  s = s + dz * dz;
  return s;
}

/* means (N,3), points (M,3) -> out (M,K) int64.  Returns 0 or 1 (bad K). */
int oracle_knn_query(int64_t N, const double *means, int64_t M,
                     const double *points, int64_t K, int64_t *out) {
  if (K < 1 || K > N) return 1;
  const int64_t keff = (K + 1 < N) ? K + 1 : N;
#pragma omp parallel
  {
    cand_t *top = (cand_t *)malloc(sizeof(cand_t) * (size_t)(keff + 1));
#pragma omp for schedule(dynamic, 64)
    for (int64_t r = 0; r < M; ++r) {
      const double *p = points + 3 * r;
      int64_t n = 0;
      /* keep the keff smallest by (d2, idx), sorted ascending */
      for (int64_t j = 0; j < N; ++j) {
        cand_t c = {sq_dist(means + 3 * j, p), j};
        if (n == keff && !cand_less(&c, &top[n - 1])) continue;
        int64_t pos = (n < keff) ? n++ : n - 1;
        while (pos > 0 && cand_less(&c, &top[pos - 1])) {
          top[pos] = top[pos - 1];
          --pos;
        }
        top[pos] = c;
      }
      int boundary_tie = (keff > K) && (sqrt(top[K - 1].d2) == sqrt(top[K].d2));
      if (!boundary_tie) {
        /* (sqrt(d2), idx) order: stable re-sort within equal-distance runs */
        int64_t a = 0;
        while (a < K) {
          int64_t b = a + 1;
          double da = sqrt(top[a].d2);
          while (b < keff && sqrt(top[b].d2) == da) ++b;
          /* run [a, b) shares one distance: order by index */
          for (int64_t i = a + 1; i < b; ++i) {
            cand_t c = top[i];
            int64_t q = i;
            while (q > a && top[q - 1].idx > c.idx) {
              top[q] = top[q - 1];
              --q;
            }
            top[q] = c;
          }
          a = b;
        }
      }
      for (int64_t k = 0; k < K; ++k) out[r * K + k] = top[k].idx;
    }
    free(top);
  }
  return 0;
}
