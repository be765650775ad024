// Warp-per-patch fused Schwarz V-cycle ("W mode"; rows a5, a6, a8 for 3D vertex
// patches whose level-1 box is at most 3 x 3 x 3, i.e. p = 3: C5).
//
// One warp owns one patch for the whole V(1,1) cycle: the patch's
// MDF-ordered ILU(0) factor M = L D L^T (reading c5) is staged ONCE into the warp's
// shared memory and serves all four triangular sweeps (pre-smoothing forward /
// backward, post-smoothing forward / backward), so the factor crosses HBM once per
// apply instead of four times (the thread-per-patch kernels of vcycle_t.cu).
//
// Sweeps as conflict-free push rounds.  With lev(k) the DAG level of node k in the
// triangular solve (longest chain of earlier neighbours), every factor entry L_ik
// (k eliminated before its neighbour i) joins k -> i with lev(k) < lev(i).
//   forward  (w = L^{-1} r):  levels ascending; in level l every k with lev(k) = l is
//            final, so all its pushes w_i -= L_ik w_k may run at once, except that two
//            pushes into the same i must not share a round.  The entries of level l
//            are packed (setup, greedy) into rounds of <= 32 entries with distinct
//            targets: one lane per entry, one __syncwarp per round.
//   backward (x = L^{-T} D^{-1} w): levels descending, x_k -= L_ik x_i with x_i final
//            once the level of i is reached; rounds of distinct targets k.
// Both directions read the same values; the backward rounds refer to them by index.
// The push form sums each node's contributions in round order instead of the
// row order of a pull sweep: identical up to rounding.
//
// Between the sweeps (lane = node): s = r_j - A x with the finest LOR rows, the
// separable restriction r_1 = P^T s, z_1 = C r_1 with C the dense operator of the
// V-cycle on levels >= 1 (reading c5 makes it symmetric; packed upper triangle of
// the fixed 3x3x3 coarse box), y = x + P z_1, s = r_j - A y; then z_j = y + M^{-1} s
// and the scatter z += I_j z_j (atomics, a8).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "patch.cuh"

namespace lorpc {

std::vector<int> tile_order(const lorpc_prec* b, int TX, int TY);  // vcycle_t.cu

// ------------------------------------------------------------------ W-record layout
// Per patch (in warp-slot order, 16-byte aligned):
//   int4 {n, nF, nB, nE}
//   rf[nF + 1], rb[nB + 1]  u16   round offsets into the forward / backward entries
//   meta[nE+1]  u16   forward entry: source k (bits 0-7) | target i (bits 8-15)
//   bvi[nE+1]   u16   backward entry -> index of its forward entry (value and nodes)
//   val[nE+1]   f64   L_ik in forward round order
//   dinv[n]     f64   1 / D_k
// Entry nE is a dummy (node n -> node n, value 0, bvi = nE): lanes past the end of
// a round apply it, so the round body needs no branch.
struct WRecLayout { int rf, rb, meta, bvi, val, dinv, total; };
__host__ __device__ __forceinline__ int a16i(int b) { return (b + 15) & ~15; }
__host__ __device__ __forceinline__ WRecLayout wrec_layout(int n, int nF, int nB, int nE) {
  WRecLayout W;
  W.rf = 16;
  W.rb = W.rf + 2 * (nF + 1);
  W.meta = a16i(W.rb + 2 * (nB + 1));
  W.bvi = a16i(W.meta + 2 * (nE + 1));
  W.val = a16i(W.bvi + 2 * (nE + 1));
  W.dinv = W.val + 8 * (nE + 1);
  W.total = a16i(W.dinv + 8 * n);
  return W;
}

constexpr int WLPMAX = 32;    // largest number of lanes per patch (entries per push round)

struct WBuildParams {
  const char* rec;            // per patch-level ILU records (schwarz.cu)
  const long long* recoff;
  const int* pord;
  int L;
  long long nslots;
  int* sizes;                 // [nslots] record bytes (pass 0; -1: scheduling failed)
  int2* rounds;               // [nslots] {nF, nB} (pass 0)
  char* wrec;                 // pass 1
  const long long* wrecoff;
  unsigned char* scratch;     // per thread, wscratch_bytes(nlmax)
  int nlmax;                  // largest nL
  int lp;                     // lanes per patch = largest round (16: two patches per warp, 32: one)
};

__host__ __device__ __forceinline__ long long wscratch_bytes(int nl) { return 8ll * nl + 4 * 256 + 2 * 258 + 16; }

// List scheduling of one sweep's push entries (e: ps[e] -> pt[e]) into rounds of at
// most lp entries with distinct targets.  An entry is eligible once its source is
// final (every push into it done in an earlier round); among the eligible entries
// the ones whose target has the longest remaining chain (height) go first.  topo =
// the push sources in a topological order.  Returns the number of rounds (-1 if the
// entries do not form a DAG); with fill, ro[] gets the round offsets and emit(p, e)
// places entry e at position p.
template <class Emit>
__device__ int wschedule(int lp, int n, int nL, const unsigned char* ps, const unsigned char* pt, const uint16_t* topo,
                         bool rev, unsigned char* indeg, unsigned char* hgt, uint16_t* ocnt, uint16_t* olist,
                         int16_t* nxt, int16_t* head, uint16_t* ro, bool fill, Emit emit) {
  for (int v = 0; v <= n; ++v) ocnt[v] = 0;
  for (int e = 0; e < nL; ++e) ocnt[ps[e] + 1]++;
  for (int v = 0; v < n; ++v) ocnt[v + 1] += ocnt[v];
  for (int v = 0; v < n; ++v) head[v] = (int16_t)ocnt[v];          // fill cursors
  for (int e = 0; e < nL; ++e) olist[head[ps[e]]++] = (uint16_t)e;
  for (int v = 0; v < n; ++v) indeg[v] = 0;
  for (int e = 0; e < nL; ++e) indeg[pt[e]]++;
  int hmax = 0;
  for (int q = n - 1; q >= 0; --q) {                                 // heights, reverse topological order
    const int v = topo[rev ? n - 1 - q : q];
    int hv = 0;
    for (int o = ocnt[v]; o < ocnt[v + 1]; ++o) hv = max(hv, hgt[pt[olist[o]]] + 1);
    hgt[v] = (unsigned char)min(hv, 255);
    hmax = max(hmax, hv);
  }
  hmax = min(hmax, 255);
  for (int b = 0; b <= hmax; ++b) head[b] = -1;
  auto release = [&](int v) {
    for (int o = ocnt[v]; o < ocnt[v + 1]; ++o) {
      const int e = olist[o];
      const int b = hgt[pt[e]];
      nxt[e] = head[b];
      head[b] = (int16_t)e;
    }
  };
  for (int v = 0; v < n; ++v) if (indeg[v] == 0) release(v);
  int done = 0, r = 0;
  int tk[WLPMAX];
  while (done < nL) {
    unsigned long long mk[4] = {0ull, 0ull, 0ull, 0ull};
    int take = 0;
    for (int b = hmax; b >= 0 && take < lp; --b) {
      int prev = -1, e = head[b];
      while (e >= 0 && take < lp) {
        const int nx = nxt[e];
        const int t = pt[e];
        if (!((mk[t >> 6] >> (t & 63)) & 1ull)) {
          mk[t >> 6] |= 1ull << (t & 63);
          tk[take++] = e;
          if (prev < 0) head[b] = (int16_t)nx; else nxt[prev] = (int16_t)nx;
        } else {
          prev = e;
        }
        e = nx;
      }
    }
    if (take == 0) return -1;
    if (fill) {
      ro[r] = (uint16_t)done;
      for (int q = 0; q < take; ++q) emit(done + q, tk[q]);
    }
    done += take;
    ++r;
    for (int q = 0; q < take; ++q) {
      const int t = pt[tk[q]];
      if (--indeg[t] == 0) release(t);
    }
  }
  if (fill) ro[r] = (uint16_t)done;
  return r;
}

// One thread per warp slot.  fill = 0: round counts and record size; fill = 1:
// write the record (layout from the pass-0 counts).
__global__ void __launch_bounds__(128) k_wrec(WBuildParams P, int fill) {
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const int nl = P.nlmax;
  unsigned char* base = P.scratch + tid * wscratch_bytes(nl);
  unsigned char* esrc = base;
  unsigned char* etgt = esrc + nl;
  unsigned char* indeg = etgt + nl;
  unsigned char* hgt = indeg + 256;
  uint16_t* olist = (uint16_t*)(((uintptr_t)(hgt + 256) + 7) & ~(uintptr_t)7);
  uint16_t* fpos = olist + nl;
  int16_t* nxt = (int16_t*)(fpos + nl);
  uint16_t* ocnt = (uint16_t*)(nxt + nl);
  int16_t* head = (int16_t*)(ocnt + 258);
  for (long long slot = tid; slot < P.nslots; slot += nthreads) {
    const long long j = P.pord[slot];
    int n = 0, nL = 0;
    const char* rec = nullptr;
    if (j >= 0) {
      rec = P.rec + P.recoff[j * P.L];
      const int4 h = *(const int4*)rec;
      n = h.x; nL = h.z;
    }
    if (n == 0) {
      if (!fill) { P.sizes[slot] = 16; P.rounds[slot] = make_int2(0, 0); }
      else *(int4*)(P.wrec + P.wrecoff[slot]) = make_int4(0, 0, 0, 0);
      continue;
    }
    const RecLayout R = rec_layout(n, nL);
    const double* D = (const double*)(rec + R.D);
    const double* Lv = (const double*)(rec + R.L);
    const uint16_t* nbv = (const uint16_t*)(rec + R.nb);
    const uint16_t* frp = (const uint16_t*)(rec + R.frp);
    const uint16_t* sch = (const uint16_t*)(rec + R.sched);
    const uint16_t* eord = (const uint16_t*)(rec + R.order);   // elimination order
    for (int t = 0; t < n; ++t)
      for (int e = frp[t]; e < frp[t + 1]; ++e) { esrc[e] = (unsigned char)nbv[e]; etgt[e] = (unsigned char)sch[t]; }
    WRecLayout W{};
    char* out = nullptr;
    if (fill) {
      const int2 nr = P.rounds[slot];
      W = wrec_layout(n, nr.x, nr.y, nL);
      out = P.wrec + P.wrecoff[slot];
      *(int4*)out = make_int4(n, nr.x, nr.y, nL);
      ((uint16_t*)(out + W.meta))[nL] = (uint16_t)(n | (n << 8));
      ((uint16_t*)(out + W.bvi))[nL] = (uint16_t)nL;
      ((double*)(out + W.val))[nL] = 0.0;
      double* dv = (double*)(out + W.dinv);
      for (int i = 0; i < n; ++i) dv[i] = 1.0 / D[i];
    }
    uint16_t* meta = fill ? (uint16_t*)(out + W.meta) : nullptr;
    uint16_t* bvi = fill ? (uint16_t*)(out + W.bvi) : nullptr;
    double* val = fill ? (double*)(out + W.val) : nullptr;
    // forward: pushes k -> i (k eliminated first), sources in elimination order
    const int nF = wschedule(P.lp, n, nL, esrc, etgt, eord, false, indeg, hgt, ocnt, olist, nxt, head,
                             fill ? (uint16_t*)(out + W.rf) : nullptr, fill != 0, [&](int p, int e) {
                               meta[p] = (uint16_t)(esrc[e] | (etgt[e] << 8));
                               val[p] = Lv[e];
                               fpos[e] = (uint16_t)p;
                             });
    // backward: pushes i -> k, sources in reverse elimination order
    const int nB = nF < 0 ? -1
                          : wschedule(P.lp, n, nL, etgt, esrc, eord, true, indeg, hgt, ocnt, olist, nxt, head,
                                      fill ? (uint16_t*)(out + W.rb) : nullptr, fill != 0,
                                      [&](int p, int e) { bvi[p] = fpos[e]; });
    if (!fill) {
      P.rounds[slot] = make_int2(nF, nB);
      P.sizes[slot] = (nF < 0 || nB < 0) ? -1 : wrec_layout(n, nF, nB, nL).total;
    }
  }
}

// packed upper triangle of the dense coarse operator on the fixed 3x3x3 box, one
// patch after another in warp-slot order (Cd: column-major n_1 x n_1 per patch)
constexpr int WNC = 27, WNPK = WNC * (WNC + 1) / 2;
__global__ void k_wpack_c(const double* __restrict__ Cd, double* __restrict__ Cq, const int* __restrict__ pord,
                          PatchGeom G, long long nslots, int ldc) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (t >= nslots * WNPK) return;
  const long long slot = t / WNPK;
  int idx = (int)(t % WNPK);
  const long long j = pord[slot];
  double v = 0.0;
  if (j >= 0) {
    int a = 0;
    while (idx >= WNC - a) { idx -= WNC - a; ++a; }
    const int bb = a + idx;
    int elo[3], ehi[3];
    patch_elems(G, j, elo, ehi);
    int ce[3];
    for (int k = 0; k < 3; ++k) ce[k] = (ehi[k] - elo[k] + 1) * (G.ml[1] - 1) - 1;
    const int ax = a % 3, ay = (a / 3) % 3, az = a / 9;
    const int bx = bb % 3, by = (bb / 3) % 3, bz = bb / 9;
    if (ax < ce[0] && ay < ce[1] && az < ce[2] && bx < ce[0] && by < ce[1] && bz < ce[2]) {
      const int n1 = ce[0] * ce[1] * ce[2];
      const int ia = ax + ce[0] * (ay + ce[1] * az), ib = bx + ce[0] * (by + ce[1] * bz);
      v = Cd[j * ldc + (long long)ia * n1 + ib];
    }
  }
  Cq[t] = v;
}

// ------------------------------------------------------------------ apply kernel
extern __shared__ __align__(16) double wsm[];

struct WParams {
  PatchGeom G;
  const double* A0;           // finest LOR level, node-major rows of 28 doubles
  const double* W;            // separable restriction tables, level 0 -> 1
  int woff[5];
  const char* wrec;
  const long long* wrecoff;   // [nslots + 1]
  const int* pord;
  long long nslots;
  const double* Cq;           // [nslots][WNPK]
  int rec_bytes;              // shared bytes reserved for a staged record
  int vec_doubles;            // per patch vector length in shared memory
  int half_doubles;           // shared doubles per patch (record + X + S)
  const double* r;
  double* z;
};

__device__ __forceinline__ void ld256w(const double* p, double& a, double& b, double& c, double& d) {
  asm("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}

// One triangular sweep as push rounds.  Forward (BWD = false): V[t] -= L V[s] for
// the entries (s -> t) of each round; backward: V[k] -= L V[i] for the entries
// reached through bvi.  Lane hl of the half-warp takes entry ro[r] + hl of round r
// (the dummy entry nE past the round's end).  The next round's entry (offsets,
// nodes, value: never written during the sweep) is loaded before the __syncwarp
// that closes the current round.  Both half-warps run nrm = max of their round
// counts (the shorter one idles on the dummy entry).
template <bool BWD>
__device__ __forceinline__ void wsweep(const uint16_t* ro, int nr, int nrm, const uint16_t* meta,
                                       const uint16_t* bvi, const double* val, int nE, double* V, int hl) {
  auto off = [&](int r) { return r <= nr ? (int)ro[r] : nE; };
  auto entry = [&](int e, int& m, double& v) {
    const int k = BWD ? bvi[e] : e;
    m = meta[k];
    v = val[k];
  };
  int b1 = off(1);
  int e0 = off(0) + hl;
  int m;
  double v;
  entry(e0 < b1 ? e0 : nE, m, v);
  int b2 = off(2);
  for (int r = 0; r < nrm; ++r) {
    const int b3 = off(r + 3);
    const int en = b1 + hl;
    int mn;
    double vn;
    entry(en < b2 ? en : nE, mn, vn);
    const int s = BWD ? (m >> 8) : (m & 255), t = BWD ? (m & 255) : (m >> 8);
    V[t] = fma(-v, V[s], V[t]);
    __syncwarp();
    m = mn; v = vn; b1 = b2; b2 = b3;
  }
}

// M^{-1} V in place: forward push rounds, D^{-1}, backward push rounds.  V[n] is the
// dummy entry's node (zero on entry).
template <int LP>
__device__ __forceinline__ void wsmooth(const char* rs, double* V, int hl) {
  const int4 h = *(const int4*)rs;
  const int n = h.x, nF = h.y, nB = h.z, nE = h.w;
  const WRecLayout W = wrec_layout(n, nF, nB, nE);
  const uint16_t* meta = (const uint16_t*)(rs + W.meta);
  const uint16_t* bvi = (const uint16_t*)(rs + W.bvi);
  const double* val = (const double*)(rs + W.val);
  const double* dinv = (const double*)(rs + W.dinv);
  const int nFm = LP == 32 ? nF : max(nF, __shfl_xor_sync(0xffffffffu, nF, 16));
  const int nBm = LP == 32 ? nB : max(nB, __shfl_xor_sync(0xffffffffu, nB, 16));
  wsweep<false>((const uint16_t*)(rs + W.rf), nF, nFm, meta, bvi, val, nE, V, hl);
  for (int i = hl; i < n; i += LP) V[i] *= dinv[i];
  __syncwarp();
  wsweep<true>((const uint16_t*)(rs + W.rb), nB, nBm, meta, bvi, val, nE, V, hl);
}

struct WBox {
  int lo[3], ext[3], cext[3], ec[3], n;
};

// Residual of the x-lines of the patch box: s = r_j - A_0 V on line (iy, iz) of each
// lane (V zero outside the box).  The 3 x 3 neighbouring lines of V are read into a
// register window once per line (columns one node ahead), so a node costs its LOR
// row (7 256-bit loads) and 27 FMAs with compile-time operands.  RESTRICT: instead
// of s, store the line's x-restriction T1[3 ln + cx] = sum_x Wx[cx][x] s_x.
constexpr int WTLX = 5;  // largest box extent (p = 3 vertex patches)
template <int LP, bool RESTRICT>
__device__ __forceinline__ void wres_lines(const WParams& P, const WBox& c, const double* __restrict__ V, double* out,
                                           const double* __restrict__ Wx, int hl) {
  const int ex = c.ext[0], ey = c.ext[1], ez = c.ext[2];
  const size_t Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const int lines = ey * ez;
  for (int ln = hl; ln < lines; ln += LP) {
    const int iy = ln % ey, iz = ln / ey;
    const size_t g0 = c.lo[0] + Nx * ((c.lo[1] + iy) + Ny * (size_t)(c.lo[2] + iz));
    const double* Lp[3][3];
    bool ok[3][3];
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        const int yy = iy + dy - 1, zz = iz + dz - 1;
        ok[dz][dy] = yy >= 0 && yy < ey && zz >= 0 && zz < ez;
        Lp[dz][dy] = V + (ok[dz][dy] ? (zz * ey + yy) * ex : 0);
      }
    double Wn[3][3][WTLX + 2];
#pragma unroll
    for (int dz = 0; dz < 3; ++dz)
#pragma unroll
      for (int dy = 0; dy < 3; ++dy) {
        Wn[dz][dy][0] = 0.0;
        Wn[dz][dy][1] = ok[dz][dy] ? Lp[dz][dy][0] : 0.0;
      }
    double res[WTLX];
    // the LOR row of node x + 1 (and its r) is loaded while node x is computed
    double an[28], rn;
#pragma unroll
    for (int d4 = 0; d4 < 7; ++d4) ld256w(P.A0 + g0 * 28 + 4 * d4, an[4 * d4], an[4 * d4 + 1], an[4 * d4 + 2], an[4 * d4 + 3]);
    rn = __ldg(P.r + g0);
#pragma unroll
    for (int x = 0; x < WTLX; ++x) {
      res[x] = 0.0;
      if (x >= ex) break;
      double av[28];
#pragma unroll
      for (int d = 0; d < 28; ++d) av[d] = an[d];
      double a0 = rn, a1 = 0.0;
      if (x + 1 < ex) {
        const double* Ar = P.A0 + (g0 + x + 1) * 28;
#pragma unroll
        for (int d4 = 0; d4 < 7; ++d4) ld256w(Ar + 4 * d4, an[4 * d4], an[4 * d4 + 1], an[4 * d4 + 2], an[4 * d4 + 3]);
        rn = __ldg(P.r + g0 + x + 1);
      }
#pragma unroll
      for (int dz = 0; dz < 3; ++dz)
#pragma unroll
        for (int dy = 0; dy < 3; ++dy)
          Wn[dz][dy][x + 2] = (ok[dz][dy] && x + 1 < ex) ? Lp[dz][dy][x + 1] : 0.0;
#pragma unroll
      for (int d = 0; d < 27; ++d) {
        const double vv = (x + 2 + dir_dx(d) <= WTLX + 1) ? Wn[dir_dz(d) + 1][dir_dy(d) + 1][x + 1 + dir_dx(d)] : 0.0;
        if (d & 1) a1 = fma(-av[d], vv, a1); else a0 = fma(-av[d], vv, a0);
      }
      res[x] = a0 + a1;
    }
    if (RESTRICT) {
#pragma unroll
      for (int cx = 0; cx < 3; ++cx) {
        double t = 0.0;
        if (cx < c.cext[0])
#pragma unroll
          for (int x = 0; x < WTLX; ++x)
            if (x < ex) t = fma(__ldg(Wx + cx * ex + x), res[x], t);
        out[3 * ln + cx] = t;
      }
    } else {
#pragma unroll
      for (int x = 0; x < WTLX; ++x)
        if (x < ex) out[ln * ex + x] = res[x];
    }
  }
}

// The coarse correction between the two smoothing steps, LP lanes per patch (lane hl
// of the patch): s = r_j - A x (x-restricted on the fly), r_1 = P^T s, z_1 = C r_1,
// X <- y = x + P z_1, S <- s = r_j - A y.  S doubles as the transfer scratch.
template <int LP>
__device__ __forceinline__ void wmid(const WParams& P, const WBox& c, double* X, double* S, bool act, long long slot,
                                     int hl) {
  const int ex = c.ext[0], ey = c.ext[1];
  const double* Wx = P.W + P.woff[c.ec[0]];
  const double* Wy = P.W + P.woff[c.ec[1]];
  const double* Wz = P.W + P.woff[c.ec[2]];
  const int ez = c.ext[2];
  // S doubles as scratch until the second residual: T1 [0,75) | T2 [75,120);
  // R1 [0,27) | Z1 [27,54) | U1 [75,120); U2 [0,75)
  double* T1 = S;
  double* T2 = S + 75;
  wres_lines<LP, true>(P, c, X, T1, Wx, hl);                            // s = r_j - A x, x-restricted
  __syncwarp();
  for (int idx = hl; idx < 9 * ez; idx += LP) {                     // y-restriction
    const int cx = idx % 3, cy = (idx / 3) % 3, zz = idx / 9;
    double acc = 0.0;
    if (cy < c.cext[1])
      for (int y = 0; y < ey; ++y) acc = fma(__ldg(Wy + cy * ey + y), T1[3 * (y + ey * zz) + cx], acc);
    T2[idx] = acc;
  }
  __syncwarp();
  double* R1 = S;
  double* Z1 = S + 27;
  for (int a = hl; a < WNC; a += LP) {                              // z-restriction: r_1 = P^T s
    const int cx = a % 3, cy = (a / 3) % 3, cz = a / 9;
    double acc = 0.0;
    if (cz < c.cext[2])
      for (int zz = 0; zz < ez; ++zz) acc = fma(__ldg(Wz + cz * ez + zz), T2[cx + 3 * (cy + 3 * zz)], acc);
    R1[a] = acc;
  }
  __syncwarp();
  if (act) {                                                         // z_1 = C r_1 (packed symmetric)
    const double* Cs = P.Cq + slot * WNPK;
    for (int a = hl; a < WNC; a += LP) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < WNC; ++b) {
        const int lo = a < b ? a : b, hi = a < b ? b : a;
        acc = fma(__ldg(Cs + lo * WNC - (lo * (lo - 1)) / 2 + (hi - lo)), R1[b], acc);
      }
      Z1[a] = acc;
    }
  }
  __syncwarp();
  double* U1 = S + 75;
  double* U2 = S;
  for (int idx = hl; idx < 9 * ez; idx += LP) {                     // z-prolongation
    const int cx = idx % 3, cy = (idx / 3) % 3, zz = idx / 9;
    double acc = 0.0;
    for (int cz = 0; cz < c.cext[2]; ++cz) acc = fma(__ldg(Wz + cz * ez + zz), Z1[cx + 3 * (cy + 3 * cz)], acc);
    U1[idx] = acc;
  }
  __syncwarp();
  for (int idx = hl; idx < 3 * ey * ez; idx += LP) {                // y-prolongation
    const int cx = idx % 3, yz = idx / 3, y = yz % ey, zz = yz / ey;
    double acc = 0.0;
    for (int cy = 0; cy < c.cext[1]; ++cy) acc = fma(__ldg(Wy + cy * ey + y), U1[cx + 3 * (cy + 3 * zz)], acc);
    U2[idx] = acc;
  }
  __syncwarp();
  for (int i = hl; i < c.n; i += LP) {                              // y = x + P z_1
    const int x = i % ex, yz = i / ex;
    double acc = 0.0;
    for (int cx = 0; cx < c.cext[0]; ++cx) acc = fma(__ldg(Wx + cx * ex + x), U2[cx + 3 * yz], acc);
    X[i] += acc;
  }
  __syncwarp();
  wres_lines<LP, false>(P, c, X, S, Wx, hl);                             // s = r_j - A y
}

// LP = 16: two patches per warp, half-warp h = lane / 16 owns slot 2 blockIdx + h;
// LP = 32: one patch per warp.
template <int LP>
__global__ void __launch_bounds__(32, LP == 32 ? 12 : 7) k_vw(WParams P) {
  constexpr int PPW = 32 / LP;
  const int lane = threadIdx.x, h = lane / LP, hl = lane & (LP - 1);
  const long long slot = PPW * (long long)blockIdx.x + h;
  const bool act = slot < P.nslots;
  char* rs = (char*)(wsm + h * P.half_doubles);
  double* X = (double*)(rs + P.rec_bytes);
  double* S = X + P.vec_doubles;
  // stage the record (one HBM pass; every later use of the factor reads shared memory)
  if (act) {
    const long long o0 = P.wrecoff[slot], o1 = P.wrecoff[slot + 1];
    const int4* src = (const int4*)(P.wrec + o0);
    int4* dst = (int4*)rs;
    const int n16 = (int)((o1 - o0) >> 4);
    for (int u = hl; u < n16; u += LP) dst[u] = __ldcs(src + u);
  } else if (hl < 5) {
    // empty slot: a valid empty record (header, round offsets and dummy entry all 0)
    ((int4*)rs)[hl] = make_int4(0, 0, 0, 0);
  }
  WBox c;
  c.n = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) { c.lo[k] = 0; c.ext[k] = 0; c.cext[k] = 0; c.ec[k] = 1; }
  if (act) {
    const long long j = P.pord[slot];
    int elo[3], ehi[3];
    patch_elems(P.G, j, elo, ehi);
    c.n = 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c.ec[k] = ehi[k] - elo[k] + 1;
      c.lo[k] = elo[k] * (P.G.ml[0] - 1) + 1;
      c.ext[k] = c.ec[k] * (P.G.ml[0] - 1) - 1;
      c.cext[k] = c.ec[k] * (P.G.ml[1] - 1) - 1;
      c.n *= c.ext[k];
    }
  }
  const int ex = c.ext[0], ey = c.ext[1];
  const size_t Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const float rex = 1.0f / max(ex, 1), rexy = 1.0f / max(ex * ey, 1);
  auto gidx = [&](int i) {
    int ix, iy, iz;
    box_xyz(i, ex, ey, rex, rexy, ix, iy, iz);
    return (c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (size_t)(c.lo[2] + iz));
  };
  for (int i = hl; i < c.n; i += LP) X[i] = __ldg(P.r + gidx(i));  // r_j = I_j^T r (a5)
  if (hl == 0) { X[c.n] = 0.0; S[c.n] = 0.0; }                      // dummy node of the sweeps
  __syncwarp();
  wsmooth<LP>(rs, X, hl);                                                // x = M^{-1} r_j
  __syncwarp();
  wmid<LP>(P, c, X, S, act, slot, hl);
  if (hl == 0) S[c.n] = 0.0;
  __syncwarp();
  wsmooth<LP>(rs, S, hl);                                                // M^{-1} s
  __syncwarp();
  for (int i = hl; i < c.n; i += LP) atomicAdd(P.z + gidx(i), X[i] + S[i]);  // z += I_j (y + M^{-1} s) (a8)
}

// ------------------------------------------------------------------ setup / apply drivers
int wrec_build(lorpc_prec* b, cudaStream_t s) {
  const long long nw = (b->J + 31) / 32, nslots = nw * 32;
  const std::vector<int> ord = tile_order(b, 32, 32);
  // W mode runs one warp per patch: the slot order is the patch order of the launch
  std::vector<int> ordw;
  ordw.reserve(ord.size());
  for (int v : ord) if (v >= 0) ordw.push_back(v);
  const long long ns = (long long)ordw.size();
  (void)nslots;
  LORPC_TRY(dalloc(&b->pord, ordw.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->pord, ordw.data(), sizeof(int) * ordw.size(), cudaMemcpyHostToDevice, s));
  int nlmax = 0;
  {
    int ext[3];
    for (int k = 0; k < 3; ++k) ext[k] = 2 * (b->lor->ml[0] - 1) - 1;
    nlmax = (int)num_edges(3, ext);
  }
  WBuildParams P{};
  P.rec = b->rec; P.recoff = b->recoff; P.pord = b->pord; P.L = b->L; P.nslots = ns; P.nlmax = nlmax;
  b->wlp = 16;
  if (const char* e = getenv("LORPC_WLP")) b->wlp = atoi(e) == 32 ? 32 : 16;
  P.lp = b->wlp;
  int dev, nsm;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev);
  const long long nthreads = std::min<long long>(ns, (long long)nsm * 512);
  const long long per = wscratch_bytes(nlmax);
  int* sizes = nullptr;
  int2* rounds = nullptr;
  LORPC_TRY(dalloc(&P.scratch, (size_t)(nthreads * per)));
  LORPC_TRY(dalloc(&sizes, (size_t)ns));
  LORPC_TRY(dalloc(&rounds, (size_t)ns));
  P.sizes = sizes; P.rounds = rounds;
  const unsigned blocks = (unsigned)((nthreads + 127) / 128);
  k_wrec<<<blocks, 128, 0, s>>>(P, 0);
  LORPC_LAUNCHED();
  std::vector<int> h((size_t)ns);
  LORPC_CUDA(cudaMemcpyAsync(h.data(), sizes, sizeof(int) * h.size(), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  if (getenv("LORPC_VERBOSE")) {
    std::vector<int2> hr((size_t)ns);
    LORPC_CUDA(cudaMemcpy(hr.data(), rounds, sizeof(int2) * hr.size(), cudaMemcpyDeviceToHost));
    double sf = 0, sb = 0, sz = 0;
    int mf = 0, mb = 0;
    for (long long i = 0; i < ns; ++i) {
      sf += hr[i].x; sb += hr[i].y; sz += h[i];
      mf = std::max(mf, hr[i].x); mb = std::max(mb, hr[i].y);
    }
    fprintf(stderr, "[lorpc] wrec: %lld patches, rounds fwd mean %.1f max %d, bwd mean %.1f max %d, record mean %.0f B\n",
            ns, sf / ns, mf, sb / ns, mb, sz / ns);
  }
  std::vector<long long> off((size_t)ns + 1);
  long long acc = 0, mx = 0;
  for (long long i = 0; i < ns; ++i) {
    if (h[i] < 0) {
      dfree(P.scratch); dfree(sizes); dfree(rounds);
      return fail(LORPC_ERR_SIZE, "wrec: push-round scheduling failed (not a DAG)");
    }
    off[i] = acc;
    acc += h[i];
    mx = std::max<long long>(mx, h[i]);
  }
  off[ns] = acc;
  b->wrec_bytes = acc;
  b->wrec_max = (int)mx;
  LORPC_TRY(dalloc(&b->wrec, (size_t)acc));
  LORPC_TRY(dalloc(&b->wrecoff, off.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->wrecoff, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, s));
  P.wrec = b->wrec; P.wrecoff = b->wrecoff;
  k_wrec<<<blocks, 128, 0, s>>>(P, 1);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(P.scratch); dfree(sizes); dfree(rounds);
  b->wslots = ns;
  // packed dense coarse operators in slot order
  LORPC_TRY(dalloc(&b->Cq, (size_t)(ns * WNPK)));
  k_wpack_c<<<nb(ns * WNPK, 256), 256, 0, s>>>(b->Cd, b->Cq, b->pord, make_geom(b), ns, b->ldc);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(b->Cd);
  return LORPC_OK;
}

static WParams make_wparams(const lorpc_prec* b, const double* r, double* z) {
  WParams P{};
  P.G = make_geom(b);
  P.A0 = b->lor->A[0];
  P.W = b->wtab;
  memcpy(P.woff, b->woff[0], sizeof(P.woff));
  P.wrec = b->wrec; P.wrecoff = b->wrecoff; P.pord = b->pord; P.nslots = b->wslots;
  P.Cq = b->Cq;
  P.rec_bytes = a16i(b->wrec_max);
  P.vec_doubles = std::max((b->max_n[0] + 2) & ~1, 120);
  P.half_doubles = P.rec_bytes / 8 + 2 * P.vec_doubles;
  P.r = r; P.z = z;
  return P;
}

size_t wmode_smem(const lorpc_prec* b) {
  return (size_t)make_wparams(b, nullptr, nullptr).half_doubles * 8 * (32 / b->wlp);
}

template <int LP>
static int launch_vw(const WParams& P, cudaStream_t s) {
  constexpr int PPW = 32 / LP;
  const size_t smem = (size_t)P.half_doubles * 8 * PPW;
  if (smem > 227 * 1024) return fail(LORPC_ERR_SIZE, "vcycle_w: patch record does not fit in shared memory");
  cudaFuncSetAttribute(k_vw<LP>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_vw<LP>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_vw<LP><<<(unsigned)((P.nslots + PPW - 1) / PPW), 32, smem, s>>>(P);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int vcycle_w_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const WParams P = make_wparams(b, r, z);
  if (P.nslots == 0) return LORPC_OK;
  return b->wlp == 32 ? launch_vw<32>(P, s) : launch_vw<16>(P, s);
}

// ================================================================== Q mode
// Fused V-cycle with LP lanes per patch (LP = 2, 4, 8; NPW = 32 / LP patches per warp)
// for structure-only orderings (natural, RCM = reading r5): the patches of a warp have
// the same free-node box, hence ONE sweep schedule (as the U-records of vcycle_t.cu).
//
// Why: the thread-per-patch kernels keep 224 patches per SM in flight (358 MB of
// factors, nothing survives in the 126 MB L2 between the four sweeps, 4 x 23 GB per
// apply on C5) and each lane's sweep is one long chain of dependent loads; the
// warp-per-patch W mode reads the factor once but fits only ~14 patches per SM.
// Q mode sits between: ~80 patches per SM (2 KB of vectors each; their factors,
// ~0.9 MB per SM, mostly stay in L2 from one sweep to the next), the factor is never
// staged whole but streams through a small cp.async ring (QD sweep steps ahead, no
// registers held by loads in flight), and the LP lanes of a patch split each column.
//
// Sweeps: column steps as in the U-records.  Step t eliminates node k(t); its column
// holds the entries L_ik of the later neighbours i, in pairs; lane hl of the patch
// owns the pairs p = hl, hl + LP, ... (at most CM per step).  Forward (push): y_i -=
// L_ik y_k for the lane's pairs, lane 0 stores x_k = y_k / D_k.  Backward (pull, steps
// descending): the lanes' partial sums of L_ik x_i meet in a shuffle reduction.  One
// __syncwarp per step.  Pairs past the column's end read zero-filled ring entries and
// the dummy node n (value 0), so a step has no branches.
//
// Per box shape (device table, shared by all warps of that shape):
//   int4 {S, E, mpmax, n}   steps, pairs per patch, widest column (pairs), nodes
//   hdr[S]          u32   node k (bits 0-7) | pairs mp (8-15) | pairs before step t (16-31)
//   idx[S][LP][CM]  u32   byte offsets 8 i0 | 8 i1 << 16 of the two nodes of pair hl + LP c
// Per warp (Q-record, 256-byte aligned):
//   int4 {shape, S, E, 0} | dinv[S][NPW] f64 | val[E NPW] f64x2: step t at pair offset
//   kp(t) NPW, then patch q at q mp(t), pairs consecutive (no padding between steps)
constexpr int QD = 4;  // sweep steps in flight in the cp.async ring

__host__ __device__ __forceinline__ int qsched_bytes(int S, int LP, int CM) { return 16 + 4 * S + 4 * S * LP * CM; }
__host__ __device__ __forceinline__ long long qrec_bytes(int S, long long E, int NPW) {
  return (16 + 8ll * S * NPW + 16ll * E * NPW + 255) & ~255ll;
}

struct QBuildParams {
  const char* rec;
  const long long* recoff;
  const int* pord;       // [nslots] patch of each slot (-1: empty)
  const int* shape_ref;  // [nshapes] reference patch of each shape
  const int* wshape;     // [warps] shape of each warp
  int L, LP, CM, nshapes;
  long long nslots;
  int4* info;            // [nshapes] {S, E, mpmax, n}
  char* sched;
  int sched_stride;
  char* qrec;
  const long long* qrecoff;
  int* bad;
};

// One thread per shape.  fill = 0: {S, E, mpmax, n} from the reference patch's record;
// fill = 1: the schedule table.
__global__ void k_qsched(QBuildParams P, int fill) {
  const int g = blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= P.nshapes) return;
  const long long j = P.shape_ref[g];
  const char* rec = P.rec + P.recoff[j * P.L];
  const int4 h = *(const int4*)rec;
  const int n = h.x, nL = h.z;
  const RecLayout R = rec_layout(n, nL);
  const uint16_t* brp = (const uint16_t*)(rec + R.brp);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const uint16_t* bkv = (const uint16_t*)(rec + R.bk);
  char* tab = P.sched + (size_t)g * P.sched_stride;
  uint32_t* hdr = (uint32_t*)(tab + 16);
  uint32_t* idx = hdr + n;
  int kp = 0, mpmax = 0;
  for (int t = 0; t < n; ++t) {
    const int b0 = brp[t], cb = brp[t + 1] - b0, mp = (cb + 1) / 2;
    mpmax = max(mpmax, mp);
    if (fill) {
      hdr[t] = (uint32_t)sch[t] | ((uint32_t)mp << 8) | ((uint32_t)kp << 16);
      for (int hl = 0; hl < P.LP; ++hl)
        for (int c = 0; c < P.CM; ++c) {
          const int pr = hl + P.LP * c;
          const int i0 = 2 * pr < cb ? bkv[b0 + 2 * pr] : n, i1 = 2 * pr + 1 < cb ? bkv[b0 + 2 * pr + 1] : n;
          idx[(t * P.LP + hl) * P.CM + c] = (uint32_t)(8 * i0) | ((uint32_t)(8 * i1) << 16);
        }
    }
    kp += mp;
  }
  if (!fill) P.info[g] = make_int4(n, kp, mpmax, n);
  else *(int4*)tab = make_int4(n, kp, mpmax, n);
}

// One thread per patch slot: checks the patch against its shape's schedule (*bad = 1
// on any difference) and writes its dinv and values into the warp's Q-record.
__global__ void __launch_bounds__(128) k_qrec(QBuildParams P) {
  const long long slot = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (slot >= P.nslots) return;
  const int NPW = 32 / P.LP;
  const long long w = slot / NPW;
  const int q = (int)(slot % NPW);
  const int g = P.wshape[w];
  const char* tab = P.sched + (size_t)g * P.sched_stride;
  const int4 ti = *(const int4*)tab;
  const int S = ti.x, E = ti.y;
  const uint32_t* hdr = (const uint32_t*)(tab + 16);
  const uint32_t* idx = hdr + S;
  char* blk = P.qrec + P.qrecoff[w];
  if (q == 0) *(int4*)blk = make_int4(g, S, E, 0);
  double* dv = (double*)(blk + 16);
  double2* val = (double2*)(blk + 16 + 8ll * S * NPW);
  const long long j = P.pord[slot];
  if (j < 0) {  // empty slot: zero factor (its vectors stay zero)
    for (int t = 0; t < S; ++t) {
      const uint32_t h = hdr[t];
      const int mp = (h >> 8) & 0xff, kp = h >> 16;
      dv[t * NPW + q] = 0.0;
      for (int pr = 0; pr < mp; ++pr) val[(size_t)kp * NPW + q * mp + pr] = make_double2(0.0, 0.0);
    }
    return;
  }
  const char* rec = P.rec + P.recoff[j * P.L];
  const int4 h4 = *(const int4*)rec;
  const int n = h4.x, nL = h4.z;
  if (n != S) { atomicExch(P.bad, 1); return; }
  const RecLayout R = rec_layout(n, nL);
  const uint16_t* brp = (const uint16_t*)(rec + R.brp);
  const uint16_t* sch = (const uint16_t*)(rec + R.sched);
  const uint16_t* bkv = (const uint16_t*)(rec + R.bk);
  const double* bLv = (const double*)(rec + R.bL);
  const double* Dn = (const double*)(rec + R.D);
  bool mism = false;
  for (int t = 0; t < S; ++t) {
    const uint32_t h = hdr[t];
    const int k = h & 0xff, mp = (h >> 8) & 0xff, kp = h >> 16;
    const int b0 = brp[t], cb = brp[t + 1] - b0;
    if (sch[t] != k || (cb + 1) / 2 != mp) { mism = true; break; }
    dv[t * NPW + q] = 1.0 / Dn[k];
    for (int pr = 0; pr < mp; ++pr) {
      const uint32_t iw = idx[(t * P.LP + pr % P.LP) * P.CM + pr / P.LP];
      const int i0 = (iw & 0xffff) >> 3, i1 = (iw >> 16) >> 3;
      double2 v;
      v.x = bLv[b0 + 2 * pr];
      if (bkv[b0 + 2 * pr] != i0) mism = true;
      if (2 * pr + 1 < cb) {
        v.y = bLv[b0 + 2 * pr + 1];
        if (bkv[b0 + 2 * pr + 1] != i1) mism = true;
      } else {
        v.y = 0.0;
      }
      val[(size_t)kp * NPW + q * mp + pr] = v;
    }
  }
  if (mism) atomicExch(P.bad, 1);
}

struct QParams {
  WParams w;
  const char* qrec;
  const long long* qrecoff;
  const char* sched;
  int sched_stride;
  int vd;                // doubles per patch vector in shared memory
};

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, uint32_t bytes) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void cp_async8(uint32_t dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
// schedule-word load that stays where it is written (a plain read-only load is sunk by
// the compiler to its first use, i.e. behind the step it is meant to overlap)
__device__ __forceinline__ uint32_t ldg_pin(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.global.nc.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// The warp's view of its Q-record and schedule during a sweep
struct QSw {
  const uint32_t* hdr;   // [S]
  const uint32_t* idx;   // [S][LP][CM], lane-adjusted (+ hl CM)
  const double* dinv;    // [S][NPW], lane-adjusted (+ q)
  const double2* val;
  int S;
  uint32_t ring_s;       // shared address of the value ring [QD][CM][32] f64x2, lane-adjusted
  uint32_t dring_s;      // shared address of the dinv ring [QD][NPW] f64, lane-adjusted
  const double2* ring;   // the same rings, generic pointers
  const double* dring;
};

// One triangular sweep of the warp's NPW patches over vector V (the lane's patch).
template <int LP, int CM, bool BWD>
__device__ __forceinline__ void qsweep(const QSw& Q, double* V, int hl, int q) {
  constexpr int NPW = 32 / LP;
  const int S = Q.S;
  char* Vb = (char*)V;
  auto T = [&](int tau) { return BWD ? S - 1 - tau : tau; };
  auto issue = [&](int tau, uint32_t h) {
    if (tau < S) {
      const int mp = (h >> 8) & 0xff, kp = h >> 16;
      const double2* src = Q.val + ((size_t)kp * NPW + q * mp);
      const uint32_t dst = Q.ring_s + (uint32_t)((tau & (QD - 1)) * CM) * 512u;
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        const int pr = hl + LP * c;
        const bool ok = pr < mp;
        cp_async16(dst + c * 512u, src + (ok ? pr : 0), ok ? 16u : 0u);
      }
      if (!BWD && hl == 0) cp_async8(Q.dring_s + (uint32_t)((tau & (QD - 1)) * NPW) * 8u, Q.dinv + T(tau) * NPW);
    }
    cp_async_commit();
  };
  if (S == 0) return;
  uint32_t hI = Q.hdr[T(0)];
#pragma unroll
  for (int tau = 0; tau < QD; ++tau) {
    const uint32_t hn = tau + 1 < S ? Q.hdr[T(tau + 1)] : 0u;
    issue(tau, hI);
    hI = hn;
  }
  uint32_t hC = Q.hdr[T(0)];
  uint32_t iC[CM];
#pragma unroll
  for (int c = 0; c < CM; ++c) iC[c] = Q.idx[T(0) * LP * CM + c];
  for (int tau = 0; tau < S; ++tau) {
    // schedule words of the next step and of the step issued next
    uint32_t hN = 0u, iN[CM];
#pragma unroll
    for (int c = 0; c < CM; ++c) iN[c] = 0u;
    if (tau + 1 < S) {
      hN = Q.hdr[T(tau + 1)];
#pragma unroll
      for (int c = 0; c < CM; ++c) iN[c] = Q.idx[T(tau + 1) * LP * CM + c];
    }
    const uint32_t hI2 = tau + QD + 1 < S ? Q.hdr[T(tau + QD + 1)] : 0u;
    cp_async_wait<QD - 1>();
    const int k8 = (hC & 0xff) * 8;
    const double2* rg = Q.ring + (tau & (QD - 1)) * CM * 32;
    double2 l[CM];
#pragma unroll
    for (int c = 0; c < CM; ++c) l[c] = rg[c * 32];
    if (!BWD) {
      const double yk = *(const double*)(Vb + k8);
      double v0[CM], v1[CM];
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        v0[c] = *(const double*)(Vb + (iC[c] & 0xffff));
        v1[c] = *(const double*)(Vb + (iC[c] >> 16));
      }
      const double dk = Q.dring[(tau & (QD - 1)) * NPW];
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        *(double*)(Vb + (iC[c] & 0xffff)) = fma(-l[c].x, yk, v0[c]);
        *(double*)(Vb + (iC[c] >> 16)) = fma(-l[c].y, yk, v1[c]);
      }
      if (hl == 0) *(double*)(Vb + k8) = yk * dk;
    } else {
      double a0 = 0.0, a1 = 0.0;
#pragma unroll
      for (int c = 0; c < CM; ++c) {
        a0 = fma(-l[c].x, *(const double*)(Vb + (iC[c] & 0xffff)), a0);
        a1 = fma(-l[c].y, *(const double*)(Vb + (iC[c] >> 16)), a1);
      }
      double a = a0 + a1;
#pragma unroll
      for (int m = 1; m < LP; m <<= 1) a += __shfl_xor_sync(0xffffffffu, a, m);
      if (hl == 0) *(double*)(Vb + k8) += a;
    }
    __syncwarp();
    issue(tau + QD, hI);
    hI = hI2;
    hC = hN;
#pragma unroll
    for (int c = 0; c < CM; ++c) iC[c] = iN[c];
  }
  cp_async_wait<0>();
}

// M^{-1} V in place (V[n] = 0 on entry: the dummy node)
template <int LP, int CM>
__device__ __forceinline__ void qsmooth(const QSw& Q, double* V, int n, int hl, int q) {
  qsweep<LP, CM, false>(Q, V, hl, q);
  if (hl == 0) V[n] = 0.0;
  __syncwarp();
  qsweep<LP, CM, true>(Q, V, hl, q);
}

template <int LP, int CM>
__global__ void __launch_bounds__(32) k_vq(QParams P) {
  constexpr int NPW = 32 / LP;
  const int lane = threadIdx.x, q = lane / LP, hl = lane & (LP - 1);
  const long long w = blockIdx.x;
  const long long slot = NPW * w + q;
  const long long j = P.w.pord[slot];
  const bool act = j >= 0;
  const char* blk = P.qrec + P.qrecoff[w];
  const int4 hd = __ldg((const int4*)blk);
  const char* tab = P.sched + (size_t)hd.x * P.sched_stride;
  const int S = hd.y;
  // shared memory: vectors [NPW][2][vd] | value ring [QD][CM][32] f64x2 | dinv ring [QD][NPW] |
  // the warp's sweep schedule (hdr[S], idx[S][LP][CM]; a global load per step would
  // stall every step on its L2 latency)
  double* X = wsm + (size_t)q * 2 * P.vd;
  double* Sv = X + P.vd;
  double2* ring = (double2*)(wsm + (size_t)NPW * 2 * P.vd);
  double* dring = (double*)(ring + QD * CM * 32);
  uint32_t* ssched = (uint32_t*)(dring + QD * NPW);
  {
    const uint32_t* gs = (const uint32_t*)(tab + 16);
    const int nwords = S * (1 + LP * CM);
    for (int i = lane; i < nwords; i += 32) ssched[i] = __ldg(gs + i);
  }
  QSw Q;
  Q.hdr = ssched;
  Q.idx = Q.hdr + S + hl * CM;
  Q.dinv = (const double*)(blk + 16) + q;
  Q.val = (const double2*)(blk + 16 + 8ll * S * NPW);
  Q.S = S;
  Q.ring = ring + lane;
  Q.dring = dring + q;
  Q.ring_s = (uint32_t)__cvta_generic_to_shared(ring + lane);
  Q.dring_s = (uint32_t)__cvta_generic_to_shared(dring + q);
  WBox c;
  c.n = 0;
#pragma unroll
  for (int k = 0; k < 3; ++k) { c.lo[k] = 0; c.ext[k] = 0; c.cext[k] = 0; c.ec[k] = 1; }
  if (act) {
    int elo[3], ehi[3];
    patch_elems(P.w.G, j, elo, ehi);
    c.n = 1;
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      c.ec[k] = ehi[k] - elo[k] + 1;
      c.lo[k] = elo[k] * (P.w.G.ml[0] - 1) + 1;
      c.ext[k] = c.ec[k] * (P.w.G.ml[0] - 1) - 1;
      c.cext[k] = c.ec[k] * (P.w.G.ml[1] - 1) - 1;
      c.n *= c.ext[k];
    }
  }
  const int ex = c.ext[0], ey = c.ext[1];
  const size_t Nx = P.w.G.Nax[0][0], Ny = P.w.G.Nax[0][1];
  const float rex = 1.0f / max(ex, 1), rexy = 1.0f / max(ex * ey, 1);
  auto gidx = [&](int i) {
    int ix, iy, iz;
    box_xyz(i, ex, ey, rex, rexy, ix, iy, iz);
    return (c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (size_t)(c.lo[2] + iz));
  };
  // r_j = I_j^T r (a5); entries past the patch (the dummy node S, empty slots) are zero
  for (int i = hl; i < P.vd; i += LP) { X[i] = i < c.n ? __ldg(P.w.r + gidx(i)) : 0.0; Sv[i] = 0.0; }
  __syncwarp();
  qsmooth<LP, CM>(Q, X, S, hl, q);                                       // x = M^{-1} r_j
  __syncwarp();
  wmid<LP>(P.w, c, X, Sv, act, slot, hl);
  if (hl == 0) Sv[S] = 0.0;
  __syncwarp();
  qsmooth<LP, CM>(Q, Sv, S, hl, q);                                      // M^{-1} s
  __syncwarp();
  for (int i = hl; i < c.n; i += LP) atomicAdd(P.w.z + gidx(i), X[i] + Sv[i]);  // z += I_j (y + M^{-1} s) (a8)
}

// Slot order of Q mode: the tile order, patches grouped by their level-0 box shape,
// each group padded to whole warps of NPW patches.  *ok = 0 when some patch differs
// from its shape's schedule (the caller falls back to the thread-mode kernels).
int qrec_build(lorpc_prec* b, cudaStream_t s, int* ok) {
  *ok = 0;
  int LP = 4;
  if (const char* e = getenv("LORPC_QLP")) LP = atoi(e);
  if (LP != 2 && LP != 4 && LP != 8) return fail(LORPC_ERR_ARG, "LORPC_QLP must be 2, 4 or 8");
  const int NPW = 32 / LP;
  const std::vector<int> ord = tile_order(b, 32, 32);
  const PatchGeom G = make_geom(b);
  std::vector<std::pair<int, std::vector<int>>> groups;  // shape key -> patches, in order of first appearance
  {
    for (int j : ord) {
      if (j < 0) continue;
      int lo[3], ext[3];
      patch_box(G, j, 0, lo, ext);
      const int key = ext[0] | (ext[1] << 10) | (ext[2] << 20);
      size_t g = 0;
      while (g < groups.size() && groups[g].first != key) ++g;
      if (g == groups.size()) groups.push_back({key, {}});
      groups[g].second.push_back(j);
    }
  }
  std::vector<int> qord, wshape, sref;
  for (size_t g = 0; g < groups.size(); ++g) {
    sref.push_back(groups[g].second[0]);
    qord.insert(qord.end(), groups[g].second.begin(), groups[g].second.end());
    qord.resize((qord.size() + NPW - 1) / NPW * NPW, -1);
    wshape.resize(qord.size() / NPW, (int)g);
  }
  const long long nslots = (long long)qord.size(), nw = nslots / NPW;
  const int nsh = (int)groups.size();
  if (nslots == 0) return LORPC_OK;
  int *d_sref = nullptr, *d_wshape = nullptr, *bad = nullptr;
  int4* d_info = nullptr;
  LORPC_TRY(dalloc(&b->pord, qord.size()));
  LORPC_TRY(dalloc(&d_sref, sref.size()));
  LORPC_TRY(dalloc(&d_wshape, wshape.size()));
  LORPC_TRY(dalloc(&d_info, (size_t)nsh));
  LORPC_TRY(dalloc(&bad, 1));
  LORPC_CUDA(cudaMemcpyAsync(b->pord, qord.data(), sizeof(int) * qord.size(), cudaMemcpyHostToDevice, s));
  LORPC_CUDA(cudaMemcpyAsync(d_sref, sref.data(), sizeof(int) * sref.size(), cudaMemcpyHostToDevice, s));
  LORPC_CUDA(cudaMemcpyAsync(d_wshape, wshape.data(), sizeof(int) * wshape.size(), cudaMemcpyHostToDevice, s));
  LORPC_CUDA(cudaMemsetAsync(bad, 0, sizeof(int), s));
  QBuildParams P{};
  P.rec = b->rec; P.recoff = b->recoff; P.pord = b->pord; P.shape_ref = d_sref; P.wshape = d_wshape;
  P.L = b->L; P.LP = LP; P.nshapes = nsh; P.nslots = nslots; P.info = d_info; P.bad = bad;
  k_qsched<<<nb(nsh, 32), 32, 0, s>>>(P, 0);
  LORPC_LAUNCHED();
  std::vector<int4> info((size_t)nsh);
  LORPC_CUDA(cudaMemcpyAsync(info.data(), d_info, sizeof(int4) * nsh, cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  int Smax = 0, mpmax = 0;
  bool fits = true;
  for (const int4& v : info) {
    Smax = std::max(Smax, v.x); mpmax = std::max(mpmax, v.z);
    if (v.y > 65535 || v.x > 254) fits = false;
  }
  // ring rows per step: the instantiated CM at or above ceil(mpmax / LP)
  const int need = std::max(1, (mpmax + LP - 1) / LP);
  int CM = 0;  // the (LP, CM) pairs vcycle_q_apply instantiates
  for (int cand : {1, 2, 3, 4, 5, 7}) {
    const bool have = LP == 2 ? (cand == 4 || cand == 5 || cand == 7) : LP == 4 ? cand <= 4 : cand <= 2;
    if (have && cand >= need) { CM = cand; break; }
  }
  auto cleanup = [&]() { dfree(d_sref); dfree(d_wshape); dfree(d_info); dfree(bad); };
  if (!fits || CM == 0) { cleanup(); dfree(b->pord); return LORPC_OK; }
  b->qlp = LP; b->qcm = CM;
  b->qsched_stride = (qsched_bytes(Smax, LP, CM) + 255) & ~255;
  LORPC_TRY(dalloc(&b->qsched, (size_t)nsh * b->qsched_stride));
  P.CM = CM; P.sched = b->qsched; P.sched_stride = b->qsched_stride;
  k_qsched<<<nb(nsh, 32), 32, 0, s>>>(P, 1);
  LORPC_LAUNCHED();
  std::vector<long long> off((size_t)nw);
  long long acc = 0;
  for (long long w = 0; w < nw; ++w) {
    off[w] = acc;
    const int4& v = info[wshape[w]];
    acc += qrec_bytes(v.x, v.y, NPW);
  }
  b->qrec_bytes = acc;
  LORPC_TRY(dalloc(&b->qrec, (size_t)acc));
  LORPC_TRY(dalloc(&b->qrecoff, off.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->qrecoff, off.data(), sizeof(long long) * off.size(), cudaMemcpyHostToDevice, s));
  P.qrec = b->qrec; P.qrecoff = b->qrecoff;
  k_qrec<<<nb(nslots, 128), 128, 0, s>>>(P);
  LORPC_LAUNCHED();
  int hbad = 0;
  LORPC_CUDA(cudaMemcpyAsync(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  cleanup();
  if (hbad) {
    dfree(b->pord); dfree(b->qrec); dfree(b->qrecoff); dfree(b->qsched);
    return LORPC_OK;
  }
  b->wslots = nslots;
  if (getenv("LORPC_VERBOSE"))
    fprintf(stderr, "[lorpc] qrec: %lld slots in %lld warps, %d shapes, LP %d, CM %d (widest column %d pairs), %.2f GB\n",
            nslots, nw, nsh, LP, CM, mpmax, acc / 1e9);
  // packed dense coarse operators in slot order
  LORPC_TRY(dalloc(&b->Cq, (size_t)(nslots * WNPK)));
  k_wpack_c<<<nb(nslots * WNPK, 256), 256, 0, s>>>(b->Cd, b->Cq, b->pord, make_geom(b), nslots, b->ldc);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(b->Cd);
  *ok = 1;
  return LORPC_OK;
}

static QParams make_qparams(const lorpc_prec* b, const double* r, double* z) {
  QParams P{};
  P.w.G = make_geom(b);
  P.w.A0 = b->lor->A[0];
  P.w.W = b->wtab;
  memcpy(P.w.woff, b->woff[0], sizeof(P.w.woff));
  P.w.pord = b->pord; P.w.nslots = b->wslots;
  P.w.Cq = b->Cq;
  P.w.r = r; P.w.z = z;
  P.qrec = b->qrec; P.qrecoff = b->qrecoff; P.sched = b->qsched; P.sched_stride = b->qsched_stride;
  P.vd = std::max((b->max_n[0] + 2) & ~1, 120);
  return P;
}

size_t qmode_smem(const lorpc_prec* b) {
  const int NPW = 32 / b->qlp;
  const int vd = std::max((b->max_n[0] + 2) & ~1, 120);
  const size_t sched = 4 * (size_t)b->max_n[0] * (1 + b->qlp * b->qcm);
  return (size_t)NPW * 2 * vd * 8 + (size_t)QD * b->qcm * 512 + (size_t)QD * NPW * 8 + ((sched + 15) & ~(size_t)15);
}

template <int LP, int CM>
static int launch_vq(const lorpc_prec* b, const QParams& P, cudaStream_t s) {
  constexpr int NPW = 32 / LP;
  const size_t smem = qmode_smem(b);
  cudaFuncSetAttribute(k_vq<LP, CM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(k_vq<LP, CM>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
  k_vq<LP, CM><<<(unsigned)(P.w.nslots / NPW), 32, smem, s>>>(P);
  LORPC_LAUNCHED();
  return LORPC_OK;
}

int vcycle_q_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const QParams P = make_qparams(b, r, z);
  if (P.w.nslots == 0) return LORPC_OK;
  if (qmode_smem(b) > 227 * 1024) return fail(LORPC_ERR_SIZE, "vcycle_q: shared memory");
  const int key = b->qlp * 16 + b->qcm;
  switch (key) {
    case 2 * 16 + 4: return launch_vq<2, 4>(b, P, s);
    case 2 * 16 + 5: return launch_vq<2, 5>(b, P, s);
    case 2 * 16 + 7: return launch_vq<2, 7>(b, P, s);
    case 4 * 16 + 1: return launch_vq<4, 1>(b, P, s);
    case 4 * 16 + 2: return launch_vq<4, 2>(b, P, s);
    case 4 * 16 + 3: return launch_vq<4, 3>(b, P, s);
    case 4 * 16 + 4: return launch_vq<4, 4>(b, P, s);
    case 8 * 16 + 1: return launch_vq<8, 1>(b, P, s);
    case 8 * 16 + 2: return launch_vq<8, 2>(b, P, s);
    default: return fail(LORPC_ERR_SIZE, "vcycle_q: (LP, CM) not compiled");
  }
}

}  // namespace lorpc
