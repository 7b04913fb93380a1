/*
 * spmv_oracle.c — C restatement of the reference's plain/vla SpMV kernels.
 * TEST INFRASTRUCTURE ONLY: used by tests/ (full-size parity checks where
 * the numpy oracle is too slow), by __graft_entry__.smoke() and as the
 * timed CPU baseline of bench.py.  The product library never links it.
 *
 * Semantics follow /root/reference/pkg/src/spmvkit/kernels.py exactly:
 *   csr_plain  kernels.py:69-82   rounded products, left-to-right row sums
 *                                  starting from the first product
 *   coo_plain  kernels.py:56-66   y = 0, then y[row] += product in storage
 *                                  order (np.add.at)
 *   dia_plain  kernels.py:85-101  y = 0, ascending diagonals, in-bounds only
 *   csr_vla    kernels.py:143-171 lane accumulators + lanes.py:107-128 tree
 * Compiled with -ffp-contract=off: no FMA, like numpy.  Pinned bit-for-bit
 * against the numpy oracle and the reference golden vectors by
 * tests/test_oracle_golden.py.
 *
 * Row-parallel loops (OpenMP) do not change any row's summation order.
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define DEFINE_KERNELS(T, SUF)                                                              \
  void oracle_csr_plain_##SUF(int64_t nrows, const uint32_t* irp, const uint32_t* aj,      \
                              const T* av, const T* x, T* y) {                              \
    _Pragma("omp parallel for schedule(dynamic, 4096)")                                     \
    for (int64_t r = 0; r < nrows; ++r) {                                                   \
      uint32_t s = irp[r], e = irp[r + 1];                                                  \
      T acc = 0;                                                                            \
      if (e > s) {                                                                          \
        acc = av[s] * x[aj[s]];                                                             \
        for (uint32_t j = s + 1; j < e; ++j) {                                              \
          T p = av[j] * x[aj[j]];                                                           \
          acc = acc + p;                                                                    \
        }                                                                                   \
      }                                                                                     \
      y[r] = acc;                                                                           \
    }                                                                                       \
  }                                                                                         \
                                                                                            \
  /* Storage-order scatter; row-sorted inputs split at row boundaries. */                   \
  void oracle_coo_plain_##SUF(int64_t nrows, int64_t nnz, const uint32_t* ai,               \
                              const uint32_t* aj, const T* av, const T* x, T* y,            \
                              int row_sorted) {                                             \
    _Pragma("omp parallel for schedule(static)")                                            \
    for (int64_t r = 0; r < nrows; ++r) y[r] = 0;                                           \
    if (!row_sorted) {                                                                      \
      for (int64_t k = 0; k < nnz; ++k) {                                                   \
        T p = av[k] * x[aj[k]];                                                             \
        y[ai[k]] = y[ai[k]] + p;                                                            \
      }                                                                                     \
      return;                                                                               \
    }                                                                                       \
    _Pragma("omp parallel")                                                                 \
    {                                                                                       \
      int nt = 1, t = 0;                                                                    \
      nt = omp_nthreads();                                                                  \
      t = omp_tid();                                                                        \
      int64_t lo = nnz * t / nt, hi = nnz * (t + 1) / nt;                                   \
      while (lo > 0 && lo < nnz && ai[lo] == ai[lo - 1]) ++lo;                              \
      while (hi > 0 && hi < nnz && ai[hi] == ai[hi - 1]) ++hi;                              \
      for (int64_t k = lo; k < hi; ++k) {                                                   \
        T p = av[k] * x[aj[k]];                                                             \
        y[ai[k]] = y[ai[k]] + p;                                                            \
      }                                                                                     \
    }                                                                                       \
  }                                                                                         \
                                                                                            \
  void oracle_dia_plain_##SUF(int64_t nrows, int64_t ncols, int64_t nd, const int32_t* offs, \
                              const T* vals, const T* x, T* y) {                            \
    _Pragma("omp parallel for schedule(static, 8192)")                                      \
    for (int64_t i = 0; i < nrows; ++i) {                                                   \
      T acc = 0;                                                                            \
      for (int64_t d = 0; d < nd; ++d) {                                                    \
        int64_t c = i + offs[d];                                                            \
        if (c >= 0 && c < ncols) {                                                          \
          T p = vals[i * nd + d] * x[c];                                                    \
          acc = acc + p;                                                                    \
        }                                                                                   \
      }                                                                                     \
      y[i] = acc;                                                                           \
    }                                                                                       \
  }                                                                                         \
                                                                                            \
  void oracle_csr_vla_##SUF(int64_t nrows, const uint32_t* irp, const uint32_t* aj,        \
                            const T* av, const T* x, T* y, int lanes) {                     \
    int width = 1;                                                                          \
    while (width < lanes) width <<= 1;                                                      \
    _Pragma("omp parallel")                                                                 \
    {                                                                                       \
      T* acc = (T*)malloc(sizeof(T) * (size_t)width);                                       \
      _Pragma("omp for schedule(dynamic, 1024)")                                            \
      for (int64_t r = 0; r < nrows; ++r) {                                                 \
        uint32_t s = irp[r], e = irp[r + 1];                                                \
        if (s == e) { y[r] = 0; continue; }                                                 \
        for (int l = 0; l < width; ++l) acc[l] = 0;                                         \
        for (uint32_t j0 = s; j0 < e; j0 += (uint32_t)lanes)                                \
          for (int l = 0; l < lanes && j0 + (uint32_t)l < e; ++l) {                         \
            T p = av[j0 + l] * x[aj[j0 + l]];                                               \
            acc[l] = acc[l] + p;                                                            \
          }                                                                                 \
        for (int w = width >> 1; w >= 1; w >>= 1)                                           \
          for (int l = 0; l < w; ++l) acc[l] = acc[l] + acc[l + w];                         \
        y[r] = acc[0];                                                                      \
      }                                                                                     \
      free(acc);                                                                            \
    }                                                                                       \
  }

#ifdef _OPENMP
#include <omp.h>
static int omp_nthreads(void) { return omp_get_num_threads(); }
static int omp_tid(void) { return omp_get_thread_num(); }
int oracle_max_threads(void) { return omp_get_max_threads(); }
void oracle_set_threads(int n) { if (n > 0) omp_set_num_threads(n); }
#else
static int omp_nthreads(void) { return 1; }
static int omp_tid(void) { return 0; }
int oracle_max_threads(void) { return 1; }
void oracle_set_threads(int n) { (void)n; }
#endif

DEFINE_KERNELS(double, f64)
DEFINE_KERNELS(float, f32)

/* matrixio.py:170-210 restricted to rows [r0, r1): row p = (z*ny+y)*nx+x,
 * neighbours in (dz, dy, dx) order (ascending columns), 26 / -1.  Two-pass:
 * irp (rebased) first, then columns and values.  Used by bench.py's
 * reference arm, which must not touch the GPU. */
static int64_t axis_cnt(int64_t n, int64_t i) { return n == 1 ? 1 : ((i == 0 || i == n - 1) ? 2 : 3); }

void oracle_stencil27_irp(int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1, uint32_t* irp) {
  irp[0] = 0;
  for (int64_t p = r0; p < r1; ++p) {
    int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
    irp[p - r0 + 1] = irp[p - r0] + (uint32_t)(axis_cnt(nx, x) * axis_cnt(ny, y) * axis_cnt(nz, z));
  }
}

void oracle_stencil27_fill_f64(int64_t nx, int64_t ny, int64_t nz, int64_t r0, int64_t r1, const uint32_t* irp,
                               uint32_t* cols, double* vals) {
  _Pragma("omp parallel for schedule(static, 4096)")
  for (int64_t p = r0; p < r1; ++p) {
    int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
    int64_t k = irp[p - r0];
    for (int dz = -1; dz <= 1; ++dz)
      for (int dy = -1; dy <= 1; ++dy)
        for (int dx = -1; dx <= 1; ++dx) {
          int64_t qx = x + dx, qy = y + dy, qz = z + dz;
          if (qx < 0 || qx >= nx || qy < 0 || qy >= ny || qz < 0 || qz >= nz) continue;
          cols[k] = (uint32_t)((qz * ny + qy) * nx + qx);
          vals[k] = (dx == 0 && dy == 0 && dz == 0) ? 26.0 : -1.0;
          ++k;
        }
  }
}
