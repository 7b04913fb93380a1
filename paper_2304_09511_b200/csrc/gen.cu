// On-device 27-point stencil generator, bit-exact with gen_stencil27
// (matrixio.py:170-210): point (x, y, z) is row (z*ny + y)*nx + x, the
// diagonal is 26, every in-grid neighbour -1, columns ascending per row.
//
// The row pointer of a point has a closed form (entries per row factor into
// per-axis neighbour counts), so every thread computes its own IRP entry
// without a scan; the 256^3 operator (449M entries) is built in
// milliseconds instead of the reference's 51 s / 36 GB of host RAM.
#include "common.cuh"

namespace spmv {

__host__ __device__ inline int64_t axis_count(int64_t n, int64_t i) {  // valid neighbours along one axis
  if (n == 1) return 1;
  return (i == 0 || i == n - 1) ? 2 : 3;
}
__host__ __device__ inline int64_t axis_prefix(int64_t n, int64_t i) {  // sum of axis_count over [0, i)
  if (n == 1) return i;
  if (i == 0) return 0;
  return 3 * i - 1 - (i == n ? 1 : 0);
}
__host__ __device__ inline int64_t stencil_irp(int64_t nx, int64_t ny, int64_t nz, int64_t p) {
  const int64_t n = nx * ny * nz;
  if (p >= n) return axis_prefix(nx, nx) * axis_prefix(ny, ny) * axis_prefix(nz, nz);
  const int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
  const int64_t sx = axis_prefix(nx, nx), sy = axis_prefix(ny, ny);
  return axis_prefix(nz, z) * sy * sx + axis_count(nz, z) * axis_prefix(ny, y) * sx +
         axis_count(nz, z) * axis_count(ny, y) * axis_prefix(nx, x);
}

template <typename T>
__global__ void stencil27_kernel(int64_t nx, int64_t ny, int64_t nz, int64_t row_begin, int64_t row_end,
                                 uint32_t* __restrict__ irp, uint32_t* __restrict__ aj, T* __restrict__ av) {
  const int64_t nloc = row_end - row_begin;
  const int64_t base = stencil_irp(nx, ny, nz, row_begin);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i <= nloc; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t p = row_begin + i;
    const int64_t o = stencil_irp(nx, ny, nz, p) - base;
    irp[i] = uint32_t(o);
    if (i == nloc) continue;
    const int64_t x = p % nx, y = (p / nx) % ny, z = p / (nx * ny);
    int64_t k = o;
    for (int dz = -1; dz <= 1; ++dz) {
      const int64_t qz = z + dz;
      if (qz < 0 || qz >= nz) continue;
      for (int dy = -1; dy <= 1; ++dy) {
        const int64_t qy = y + dy;
        if (qy < 0 || qy >= ny) continue;
        for (int dx = -1; dx <= 1; ++dx) {
          const int64_t qx = x + dx;
          if (qx < 0 || qx >= nx) continue;
          aj[k] = uint32_t((qz * ny + qy) * nx + qx);
          av[k] = (dx == 0 && dy == 0 && dz == 0) ? T(26.0) : T(-1.0);
          ++k;
        }
      }
    }
  }
}

}  // namespace spmv

using namespace spmv;

extern "C" {

int spmv_stencil27_nnz(int64_t nx, int64_t ny, int64_t nz, int64_t* nnz_out) {
  if (!nnz_out) return fail(SPMV_INVALID_ARG, "nnz_out is NULL");
  if (nx < 1 || ny < 1 || nz < 1) return fail(SPMV_INVALID_ARG, "grid dimensions must be >= 1");
  const double n = double(nx) * double(ny) * double(nz);
  if (n > 4294967295.0 || 27.0 * n > 4294967295.0)
    return fail(SPMV_INDEX_OVERFLOW, "%lldx%lldx%lld grid exceeds 32-bit indexing", (long long)nx, (long long)ny,
                (long long)nz);
  *nnz_out = axis_prefix(nx, nx) * axis_prefix(ny, ny) * axis_prefix(nz, nz);
  return SPMV_OK;
}

int spmv_stencil27_fill(int dtype, int64_t nx, int64_t ny, int64_t nz, int64_t row_begin, int64_t row_end,
                        uint32_t* irp, uint32_t* aj, void* av, void* stream) {
  if (!valid_dtype(dtype)) return fail(SPMV_INVALID_ARG, "unsupported dtype %d", dtype);
  int64_t nnz = 0;
  int rc = spmv_stencil27_nnz(nx, ny, nz, &nnz);
  if (rc) return rc;
  const int64_t n = nx * ny * nz;
  if (row_begin < 0 || row_end < row_begin || row_end > n) return fail(SPMV_INVALID_ARG, "bad row range");
  if (!irp) return fail(SPMV_INVALID_ARG, "row_pointers_out is NULL");
  cudaStream_t st = as_stream(stream);
  const int64_t work = row_end - row_begin + 1;
  int64_t grid = (work + 255) / 256;
  const int64_t cap = int64_t(sm_count()) * 32;
  if (grid > cap) grid = cap;
  if (dtype == SPMV_F64)
    stencil27_kernel<double><<<unsigned(grid), 256, 0, st>>>(nx, ny, nz, row_begin, row_end, irp, aj,
                                                              static_cast<double*>(av));
  else
    stencil27_kernel<float><<<unsigned(grid), 256, 0, st>>>(nx, ny, nz, row_begin, row_end, irp, aj,
                                                             static_cast<float*>(av));
  SPMV_LAUNCH_CHECK();
  return SPMV_OK;
}

}  // extern "C"
