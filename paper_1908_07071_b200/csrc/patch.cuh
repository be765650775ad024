// Patch geometry, ILU record layout and grid helpers shared by the Schwarz
// setup (schwarz.cu) and apply (vcycle.cu) translation units.
#pragma once
#include "device.cuh"

namespace lorpc {

// ------------------------------------------------------------------ patch geometry
struct PatchGeom {
  int d, kind;          // kind 0 vertex, 1 star, 2 single patch (B(1))
  int n[3];             // elements per axis
  int ml[MAXL];         // nodes per element per axis at each level
  int Nax[MAXL][3];     // level grid per axis
  int L;
  int vz0;              // vertex patches: z index of the first patch plane (slab subsets)
  const short* erng;    // per patch element ranges {elo0, ehi0, elo1, ehi1, elo2, ehi2} (extended
                        // vertex patches, reading r6) or nullptr (default ranges)
};

__host__ __device__ __forceinline__ void patch_elems(const PatchGeom& G, long long j, int* elo, int* ehi) {
  if (G.erng) {
    for (int k = 0; k < 3; ++k) { elo[k] = G.erng[6 * j + 2 * k]; ehi[k] = G.erng[6 * j + 2 * k + 1]; }
    return;
  }
  if (G.kind == 2) {  // single patch B(1): the whole domain
    for (int k = 0; k < 3; ++k) { elo[k] = 0; ehi[k] = k < G.d ? G.n[k] - 1 : 0; }
    return;
  }
  if (G.kind == 0) {
    const long long nv0 = G.n[0] + 1, nv1 = G.n[1] + 1;
    const int v[3] = {(int)(j % nv0), (int)((j / nv0) % nv1), (int)(j / (nv0 * nv1)) + G.vz0};
    for (int k = 0; k < 3; ++k) {
      if (k >= G.d) { elo[k] = ehi[k] = 0; continue; }
      elo[k] = v[k] - 1 < 0 ? 0 : v[k] - 1;
      ehi[k] = v[k] < G.n[k] - 1 ? v[k] : G.n[k] - 1;
    }
  } else {
    const int e[3] = {(int)(j % G.n[0]), (int)((j / G.n[0]) % G.n[1]), (int)(j / ((long long)G.n[0] * G.n[1]))};
    for (int k = 0; k < 3; ++k) {
      if (k >= G.d) { elo[k] = ehi[k] = 0; continue; }
      elo[k] = e[k] - 1 < 0 ? 0 : e[k] - 1;
      ehi[k] = e[k] + 1 < G.n[k] - 1 ? e[k] + 1 : G.n[k] - 1;
    }
  }
}
// free node box at level l: first free node lo[k] (level-global), extent ext[k]
__host__ __device__ __forceinline__ void patch_box(const PatchGeom& G, long long j, int l, int* lo, int* ext) {
  int elo[3], ehi[3];
  patch_elems(G, j, elo, ehi);
  const int m = G.ml[l];
  for (int k = 0; k < 3; ++k) {
    if (k >= G.d) { lo[k] = 0; ext[k] = 1; continue; }
    lo[k] = elo[k] * (m - 1) + 1;
    ext[k] = (ehi[k] - elo[k] + 1) * (m - 1) - 1;
  }
}
__host__ __device__ __forceinline__ long long num_edges(int d, const int* ext) {
  // half-stencil directions: lexicographically positive offsets
  long long s = 0;
  for (int dz = (d == 3 ? -1 : 0); dz <= (d == 3 ? 1 : 0); ++dz)
    for (int dy = -1; dy <= 1; ++dy)
      for (int dx = -1; dx <= 1; ++dx) {
        const bool pos = dz > 0 || (dz == 0 && (dy > 0 || (dy == 0 && dx > 0)));
        if (!pos) continue;
        long long c = 1;
        const int o[3] = {dx, dy, dz};
        for (int k = 0; k < d; ++k) { int v = ext[k] - (o[k] < 0 ? -o[k] : o[k]); c *= v > 0 ? v : 0; }
        s += c;
      }
  return s;
}
__host__ __device__ __forceinline__ long long a8(long long b) { return (b + 7) & ~7ll; }
// Per patch-level ILU record.  Rows are stored in schedule order t (DAG levels
// of the triangular solves, ties in elimination order):
//   D[n]      pivots (natural index)
//   L[nL]     lower entries L_ij of row sched[t], rows consecutive (forward sweep)
//   fnbr[nL]  natural index j of each L entry
//   frow[n+1] row pointers into L / fnbr
//   bent[nL]  backward entries of row sched[t]: (k | pos << 16) with L[pos] = L_ki
//   brow[n+1] row pointers into bent
//   sched[n], lptr[n+1] (DAG level pointers), order[n] (elimination order)
// Per patch-level ILU record (M = L D L^T).  The off-diagonal entries are stored
// once, in forward-solve order: grouped by DAG level of the triangular solve,
// within a level by row (schedule order), within a row by direction:
//   D[n]        pivots (natural index)
//   L[nL], nb[nL]   forward entries L_ij and columns j, rows in schedule order
//   bL[nL], bk[nL]  backward (L^T) entries of row i: L_ki (value duplicated, so no
//                   load depends on another) and the later neighbour k
//   frp[n+1], brp[n+1]  entry offsets of the row sched[t] (forward / backward)
//   lptr[n+1]   DAG level row pointers into sched;  sched[n] rows (natural index)
//   order[n]    elimination order (export only)
// Each lane sweeps whole rows (row-per-lane, rows of one DAG level in parallel).
struct RecLayout { long long D, L, nb, bL, bk, frp, brp, lptr, sched, order, total; };
__host__ __device__ __forceinline__ RecLayout rec_layout(int n, long long nL) {
  RecLayout R;
  R.D = 16;
  R.L = R.D + 8ll * n;
  R.nb = R.L + 8ll * nL;
  R.bL = R.nb + a8(2ll * nL);
  R.bk = R.bL + 8ll * nL;
  R.frp = R.bk + a8(2ll * nL);
  R.brp = R.frp + a8(2ll * (n + 1));
  R.lptr = R.brp + a8(2ll * (n + 1));
  R.sched = R.lptr + a8(2ll * (n + 1));
  R.order = R.sched + a8(2ll * n);
  R.total = (R.order + 2ll * n + 15) & ~15ll;  // 16-byte aligned patch records
  return R;
}


// floor(i / d) for 0 <= i < 2^20 and small d, from a precomputed float 1/d
// (margin 0.5/d against the float rounding of (i + 0.5)/d): avoids the ~20-
// instruction integer division in the per-node index arithmetic.
__device__ __forceinline__ int qdiv(int i, float rd) { return __float2int_rz(((float)i + 0.5f) * rd); }
// (x, y, z) of a box index i in an ex x ey x ez box
__device__ __forceinline__ void box_xyz(int i, int ex, int ey, float rex, float rexy, int& x, int& y, int& z) {
  z = qdiv(i, rexy);
  const int r = i - z * ex * ey;
  y = qdiv(r, rex);
  x = r - y * ex;
}

template <int DIM>
__device__ __forceinline__ int doff(int d, int ex, int ey) {
  return dir_dx(d) + ex * (dir_dy(d) + ey * (DIM == 3 ? dir_dz(d) : 0));
}

template <int DIM>
__device__ __forceinline__ bool interior_of(long long g, int3 Nv, int* c) {
  c[0] = (int)(g % Nv.x); c[1] = (int)((g / Nv.x) % Nv.y); c[2] = (int)(g / ((long long)Nv.x * Nv.y));
  bool in = c[0] > 0 && c[0] < Nv.x - 1 && c[1] > 0 && c[1] < Nv.y - 1;
  if (DIM == 3) in = in && c[2] > 0 && c[2] < Nv.z - 1;
  return in;
}
template <int DIM>
__device__ __forceinline__ double stencil_apply(const double* A, const double* z, long long g, int3 Nv, long long NT) {
  constexpr int ND = Dirs<DIM>::ND;
  double acc = 0.0;
  for (int d = 0; d < ND; ++d) {
    const long long o = dir_dx(d) + (long long)Nv.x * (dir_dy(d) + (long long)Nv.y * (DIM == 3 ? dir_dz(d) : 0));
    acc += A[g * Dirs<DIM>::NDP + d] * z[g + o];
  }
  return acc;
}
// mode 0: z = r / d ; s = (later) ;  mode 1: s = r - A z ; mode 2: z += (r - A z)/d written to s then copied

static inline unsigned nb(long long n, int t) { return (unsigned)((n + t - 1) / t); }
static inline int3 i3(const int* a) { return make_int3(a[0], a[1], a[2]); }
PatchGeom make_geom(const lorpc_prec* b);

}  // namespace lorpc
