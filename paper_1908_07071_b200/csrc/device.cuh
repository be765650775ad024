// Device helpers shared by the lorpc kernels.
#pragma once
#include "common.h"

namespace lorpc {

// Multilinear element map of element (ex,ey,ez): x(xi), J = dx/dxi (row-major [i][k]).
template <int DIM>
__device__ __forceinline__ void elem_map(const double* __restrict__ V, const int* nv, int ex, int ey, int ez,
                                         const double* xi, double* x, double* J) {
#pragma unroll
  for (int i = 0; i < DIM; ++i) {
    x[i] = 0.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) J[i * DIM + k] = 0.0;
  }
#pragma unroll
  for (int c = 0; c < (1 << DIM); ++c) {
    const int cx = c & 1, cy = (c >> 1) & 1, cz = (c >> 2) & 1;
    long long vid = (ex + cx) + (long long)nv[0] * ((ey + cy) + (long long)nv[1] * (DIM == 3 ? ez + cz : 0));
    double ph[3], dph[3];
    const int cb[3] = {cx, cy, cz};
#pragma unroll
    for (int k = 0; k < DIM; ++k) { ph[k] = cb[k] ? xi[k] : 1.0 - xi[k]; dph[k] = cb[k] ? 1.0 : -1.0; }
    double s = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) s *= ph[k];
#pragma unroll
    for (int i = 0; i < DIM; ++i) {
      const double v = V[vid * DIM + i];
      x[i] += v * s;
#pragma unroll
      for (int k = 0; k < DIM; ++k) {
        double g = dph[k];
#pragma unroll
        for (int m = 0; m < DIM; ++m) if (m != k) g *= ph[m];
        J[i * DIM + k] += v * g;
      }
    }
  }
}

template <int DIM>
__device__ __forceinline__ double inv_det(const double* J, double* Ji) {
  if (DIM == 2) {
    double det = J[0] * J[3] - J[1] * J[2];
    double r = 1.0 / det;
    Ji[0] = J[3] * r; Ji[1] = -J[1] * r; Ji[2] = -J[2] * r; Ji[3] = J[0] * r;
    return det;
  } else {
    double c0 = J[4] * J[8] - J[5] * J[7], c1 = J[5] * J[6] - J[3] * J[8], c2 = J[3] * J[7] - J[4] * J[6];
    double det = J[0] * c0 + J[1] * c1 + J[2] * c2;
    double r = 1.0 / det;
    Ji[0] = c0 * r; Ji[1] = (J[2] * J[7] - J[1] * J[8]) * r; Ji[2] = (J[1] * J[5] - J[2] * J[4]) * r;
    Ji[3] = c1 * r; Ji[4] = (J[0] * J[8] - J[2] * J[6]) * r; Ji[5] = (J[2] * J[3] - J[0] * J[5]) * r;
    Ji[6] = c2 * r; Ji[7] = (J[1] * J[6] - J[0] * J[7]) * r; Ji[8] = (J[0] * J[4] - J[1] * J[3]) * r;
    return det;
  }
}

// 3^d stencil direction helpers: dir = (dx+1) + 3(dy+1) [+ 9(dz+1)]
// LOR stencil matrices are stored node-major, NDP doubles per node (the ND
// coefficients and a zero pad to a 16-byte multiple), so that one node's row is
// contiguous and 16-byte aligned.
template <int DIM> struct Dirs {
  static constexpr int ND = DIM == 2 ? 9 : 27;
  static constexpr int NDP = DIM == 2 ? 10 : 28;
  static constexpr int CENTER = (ND - 1) / 2;
};
__host__ __device__ __forceinline__ int ndp_of(int dim) { return dim == 2 ? 10 : 28; }
__host__ __device__ __forceinline__ int dir_dx(int d) { return d % 3 - 1; }
__host__ __device__ __forceinline__ int dir_dy(int d) { return (d / 3) % 3 - 1; }
__host__ __device__ __forceinline__ int dir_dz(int d) { return d / 9 - 1; }

// bitmask of directions whose neighbour lies inside a box [0,ex)x[0,ey)x[0,ez)
template <int DIM>
__device__ __forceinline__ uint32_t exist_mask(int ix, int iy, int iz, int ex, int ey, int ez) {
  // per-axis masks of directions with d = -1 / +1
  constexpr uint32_t XM = DIM == 2 ? 0x049u : 0x1249249u;      // dx = -1
  constexpr uint32_t XP = DIM == 2 ? 0x124u : 0x4924924u;      // dx = +1
  constexpr uint32_t YM = DIM == 2 ? 0x007u : 0x01C0E07u;      // dy = -1
  constexpr uint32_t YP = DIM == 2 ? 0x1C0u : 0x70381C0u;      // dy = +1
  constexpr uint32_t ZM = 0x00001FFu, ZP = 0x7FC0000u;
  constexpr uint32_t FULL = DIM == 2 ? 0x1FFu : 0x7FFFFFFu;
  uint32_t m = FULL;
  if (ix == 0) m &= ~XM;
  if (ix == ex - 1) m &= ~XP;
  if (iy == 0) m &= ~YM;
  if (iy == ey - 1) m &= ~YP;
  if (DIM == 3) {
    if (iz == 0) m &= ~ZM;
    if (iz == ez - 1) m &= ~ZP;
  }
  return m;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace lorpc
