// Thread-per-patch Schwarz V-cycle (rows a5, a6, a8; "patches are
// processed independently and batched").
//
// One lane owns one patch, one warp owns 32 consecutive patches.  The MDF-ordered
// ILU(0) sweeps, a strictly sequential chain per patch, run lane-parallel over
// the warp's 32 patches with no synchronisation and no reductions: lane q walks
// its own patch's rows in elimination-schedule order.  The factors are stored
// warp-interleaved ("T-records", built from the per-patch records at setup) so
// that every load of a sweep step is one coalesced 256-byte row; the step is
// padded to the warp's widest row and the padding lanes are predicated off (no
// memory traffic).  The stencil phases (gather, residual, transfers, dense coarse
// operator, scatter) are cooperative: all 32 lanes work on one patch at a time.
//
// Shared memory per warp: vector X of the 32 patches is laid out [node][patch]
// with an XOR swizzle, element (i, q) at X + 32 i + (q ^ (i & 15)), so that both
// the sweeps (lanes = patches, arbitrary rows) and the cooperative phases (lanes
// = consecutive nodes of one patch) are free of bank conflicts within a
// half-warp (the sweeps up to the random row collisions of the MDF orderings).
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "patch.cuh"

namespace lorpc {

// ------------------------------------------------------------------ T-records
// Block of (warp w, level 0) at trecoff[w], 256-byte aligned:
//   int4 {S, Kf, Kb, 0}: S steps (largest patch of the warp), Kf / Kb entry slots
//   hdr[S][32] u32   VO(node) | cf << 16 | cb << 24 of the row of step t (schedule order)
//   D[S][32]   f64   its pivot
//   Lf[Kf/2][32][2] f64, Lb[Kb/2][32][2] f64   forward L_ij / backward L_ki, in
//                    entry pairs (one 16-byte load per lane and pair)
//   Cf[Kf/2][32][2] u16, Cb[Kb/2][32][2] u16   VO of their neighbour node j / k
// Step t of the forward sweep owns the pair rows [sum_{t'<t} mp_t', + mp_t) with
// mp_t = max over the warp's lanes of ceil(cf / 2); the backward sweep likewise.
// Shared-memory layout of the warp's 32 patch vectors: node i of patch (lane) q at
// word VO(i, q) = 33 i + q, conflict-free for lanes = patches at one node and for
// lanes = consecutive nodes of one patch.  The T-records store these word offsets
// (lane-specific) instead of node numbers.
#define VO(i, q) ((i) * 33 + (q))
struct TRecLayout { long long hdr, D, Lf, Lb, Cf, Cb, total; };
__host__ __device__ __forceinline__ long long a256(long long b) { return (b + 255) & ~255ll; }
__host__ __device__ __forceinline__ TRecLayout trec_layout(int S, int Kf, int Kb) {
  TRecLayout T;
  T.hdr = 256;
  T.D = a256(T.hdr + 128ll * S);
  T.Lf = T.D + 256ll * S;
  T.Lb = T.Lf + 256ll * Kf;
  T.Cf = T.Lb + 256ll * Kb;
  T.Cb = T.Cf + 64ll * Kf;
  T.total = a256(T.Cb + 64ll * Kb);
  return T;
}

struct TRecParams {
  const char* rec;
  const long long* recoff;
  long long J;
  int L, Ld;
  int dummy[MAXL];
  long long* sizes;
  char* trec;
  const long long* trecoff;
};

// fill = 0: block sizes; fill = 1: write the blocks.  Thread = patch.
__global__ void __launch_bounds__(128) k_trec(TRecParams P, int fill) {
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long w = j >> 5;
  const int lane = threadIdx.x & 31;
  if ((w << 5) >= P.J) return;  // warp-uniform
  for (int l = 0; l < P.Ld; ++l) {
    int n = 0, nL = 0;
    const char* rec = P.rec;
    if (j < P.J) {
      rec = P.rec + P.recoff[j * P.L + l];
      const int4 h = *(const int4*)rec;
      n = h.x; nL = h.z;
    }
    const RecLayout R = rec_layout(n, nL);
    const uint16_t* frp = (const uint16_t*)(rec + R.frp);
    const uint16_t* brp = (const uint16_t*)(rec + R.brp);
    const int S = (int)__reduce_max_sync(0xffffffffu, (unsigned)n);
    int Kf = 0, Kb = 0;
    for (int t = 0; t < S; ++t) {
      const unsigned cf = t < n ? frp[t + 1] - frp[t] : 0u, cb = t < n ? brp[t + 1] - brp[t] : 0u;
      Kf += 2 * (int)__reduce_max_sync(0xffffffffu, (cf + 1) / 2);
      Kb += 2 * (int)__reduce_max_sync(0xffffffffu, (cb + 1) / 2);
    }
    const TRecLayout T = trec_layout(S, Kf, Kb);
    if (!fill) {
      if (lane == 0) P.sizes[w * P.Ld + l] = T.total;
      continue;
    }
    char* blk = P.trec + P.trecoff[w * P.Ld + l];
    if (lane == 0) *(int4*)blk = make_int4(S, Kf, Kb, 0);
    uint32_t* H = (uint32_t*)(blk + T.hdr);
    double* Dd = (double*)(blk + T.D);
    double* Lf = (double*)(blk + T.Lf);
    double* Lb = (double*)(blk + T.Lb);
    uint16_t* Cf = (uint16_t*)(blk + T.Cf);
    uint16_t* Cb = (uint16_t*)(blk + T.Cb);
    const double* Dn = (const double*)(rec + R.D);
    const double* Lv = (const double*)(rec + R.L);
    const uint16_t* nbv = (const uint16_t*)(rec + R.nb);
    const double* bLv = (const double*)(rec + R.bL);
    const uint16_t* bkv = (const uint16_t*)(rec + R.bk);
    const uint16_t* sch = (const uint16_t*)(rec + R.sched);
    const int dummy = VO(P.dummy[l], lane);
    int kf = 0, kb = 0;
    for (int t = 0; t < S; ++t) {
      int node = dummy, f0 = 0, b0 = 0;
      unsigned cf = 0, cb = 0;
      double dv = 1.0;
      if (t < n) {
        node = VO(sch[t], lane);
        f0 = frp[t]; cf = frp[t + 1] - f0;
        b0 = brp[t]; cb = brp[t + 1] - b0;
        dv = Dn[sch[t]];
      }
      H[t * 32 + lane] = (uint32_t)node | (cf << 16) | (cb << 24);
      Dd[t * 32 + lane] = dv;
      const int mf = 2 * (int)__reduce_max_sync(0xffffffffu, (cf + 1) / 2);
      for (int k = 0; k < mf; ++k) {
        const bool in = k < (int)cf;
        const long long ix = ((long long)(kf + k) / 2 * 32 + lane) * 2 + (k & 1);
        Lf[ix] = in ? Lv[f0 + k] : 0.0;
        Cf[ix] = (uint16_t)(in ? VO(nbv[f0 + k], lane) : dummy);
      }
      kf += mf;
      const int mb = 2 * (int)__reduce_max_sync(0xffffffffu, (cb + 1) / 2);
      for (int k = 0; k < mb; ++k) {
        const bool in = k < (int)cb;
        const long long ix = ((long long)(kb + k) / 2 * 32 + lane) * 2 + (k & 1);
        Lb[ix] = in ? bLv[b0 + k] : 0.0;
        Cb[ix] = (uint16_t)(in ? VO(bkv[b0 + k], lane) : dummy);
      }
      kb += mb;
    }
  }
}

// Cdi[w][k][q] = Cd[32 w + q][k] (zero for q beyond J)
__global__ void k_interleave_c(const double* __restrict__ Cd, double* __restrict__ Cdi, long long J, int ldc) {
  const long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long nw = (J + 31) / 32;
  if (t >= nw * 32 * ldc) return;
  const int q = (int)(t % 32);
  const long long k = (t / 32) % ldc, w = t / (32ll * ldc);
  const long long j = w * 32 + q;
  Cdi[t] = j < J ? Cd[j * ldc + k] : 0.0;
}

int trec_build(lorpc_prec* b, cudaStream_t s) {
  const long long nw = (b->J + 31) / 32;
  const int Ld = 1;  // T-records of the finest level only (thread mode requires Ld == 1)
  TRecParams P{};
  P.rec = b->rec; P.recoff = b->recoff; P.J = b->J; P.L = b->L; P.Ld = Ld;
  for (int l = 0; l < b->L; ++l) P.dummy[l] = b->max_n[l];
  long long* sizes = nullptr;
  LORPC_TRY(dalloc(&sizes, (size_t)(nw * Ld)));
  P.sizes = sizes;
  const unsigned blocks = (unsigned)((nw * 32 + 127) / 128);
  k_trec<<<blocks, 128, 0, s>>>(P, 0);
  LORPC_LAUNCHED();
  std::vector<long long> h((size_t)(nw * Ld));
  LORPC_CUDA(cudaMemcpyAsync(h.data(), sizes, sizeof(long long) * h.size(), cudaMemcpyDeviceToHost, s));
  LORPC_CUDA(cudaStreamSynchronize(s));
  long long off = 0;
  for (auto& v : h) { const long long sz = v; v = off; off += sz; }
  b->trec_bytes = off;
  LORPC_TRY(dalloc(&b->trec, (size_t)off));
  LORPC_TRY(dalloc(&b->trecoff, h.size()));
  LORPC_CUDA(cudaMemcpyAsync(b->trecoff, h.data(), sizeof(long long) * h.size(), cudaMemcpyHostToDevice, s));
  P.trec = b->trec; P.trecoff = b->trecoff;
  k_trec<<<blocks, 128, 0, s>>>(P, 1);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(sizes);
  // dense coarse operators interleaved by patch within each warp; r_1 / z_1 scratch
  LORPC_TRY(dalloc(&b->Cdi, (size_t)(nw * 32 * b->ldc)));
  k_interleave_c<<<nb(nw * 32 * b->ldc, 256), 256, 0, s>>>(b->Cd, b->Cdi, b->J, b->ldc);
  LORPC_LAUNCHED();
  LORPC_CUDA(cudaStreamSynchronize(s));
  dfree(b->Cd);
  LORPC_TRY(dalloc(&b->zpark, (size_t)(nw * (3 * b->max_n[0] + 2 * b->max_n[1]) * 32)));
  return LORPC_OK;
}

// ------------------------------------------------------------------ kernel
extern __shared__ __align__(16) double tsm[];

struct TcParams {
  PatchGeom G;
  const double* A0;  // finest LOR level, node-major rows of NDP doubles
  const double* W;   // separable restriction tables, level 0 -> 1
  int woff[4];
  const char* trec;
  const long long* trecoff;
  long long J;
  const double* Cd;  // [warps][ldc][32] dense operator of the V-cycle on levels >= 1 (Ld = 1), lane q's
  int ldc;           //   column-major n1 x n1 matrix interleaved by patch
  double *xpark, *ypark, *spark;  // [warps][n0max][32] x, y, s of the warp's patches (lane columns)
  double* rz;        // [warps][2][n1max][32] r_1, z_1
  int n1max;
  int n0max;         // largest finest-level patch (= the dummy node index)
  int tpoff;         // the warp's 32 patch geometries (TPatch)
  int pfd;                        // L2 prefetch distance of the sweeps (pair rows)
  int warp_doubles;
  const double* r;
  double* z;
};

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}


// One sweep step's factor data, register-resident (NP = max entry pairs per row)
template <int NP>
struct TStage {
  double2 l[NP];
  uint32_t c[NP];
};
// Loads of one step: mp pair rows (warp-uniform) from row kp.  Lanes whose row
// is shorter skip the value loads of their padding pairs (no memory traffic);
// their stale register values meet the zero at the dummy node in tdot, so the
// stage must start finite (zeroed).  The neighbour offsets are always loaded
// (padding holds the dummy).  Entered by a jump into a fall-through sequence
// instead of one branch per pair.
#define LORPC_TL_PAIR(P_)                                            \
  if ((P_) < NP) {                                                   \
    constexpr int pp = (P_) < NP ? (P_) : 0;                         \
    if (2 * pp < cnt) s.l[pp] = __ldcs(Lq + pp * 32);                \
    s.c[pp] = __ldcs(Cq + pp * 32);                                  \
  }
template <int NP>
__device__ __forceinline__ void tload(TStage<NP>& s, const double2* __restrict__ Lp, const uint32_t* __restrict__ Cp,
                                      int kp, int mp, int cnt) {
  const double2* Lq = Lp + (long long)kp * 32;
  const uint32_t* Cq = Cp + (long long)kp * 32;
  switch (mp) {
    case 13: LORPC_TL_PAIR(12); [[fallthrough]];
    case 12: LORPC_TL_PAIR(11); [[fallthrough]];
    case 11: LORPC_TL_PAIR(10); [[fallthrough]];
    case 10: LORPC_TL_PAIR(9); [[fallthrough]];
    case 9: LORPC_TL_PAIR(8); [[fallthrough]];
    case 8: LORPC_TL_PAIR(7); [[fallthrough]];
    case 7: LORPC_TL_PAIR(6); [[fallthrough]];
    case 6: LORPC_TL_PAIR(5); [[fallthrough]];
    case 5: LORPC_TL_PAIR(4); [[fallthrough]];
    case 4: LORPC_TL_PAIR(3); [[fallthrough]];
    case 3: LORPC_TL_PAIR(2); [[fallthrough]];
    case 2: LORPC_TL_PAIR(1); [[fallthrough]];
    case 1: LORPC_TL_PAIR(0); [[fallthrough]];
    default: break;
  }
}
#undef LORPC_TL_PAIR
#define LORPC_TD_PAIR(P_)                                            \
  if ((P_) < NP) {                                                   \
    constexpr int pp = (P_) < NP ? (P_) : 0;                         \
    a0 -= s.l[pp].x * tsm[X + (s.c[pp] & 0xffff)];                   \
    a1 -= s.l[pp].y * tsm[X + (s.c[pp] >> 16)];                      \
  }
template <int NP>
__device__ __forceinline__ double tdot(const TStage<NP>& s, int mp, double a0, int X) {
  double a1 = 0.0;
  switch (mp) {
    case 13: LORPC_TD_PAIR(12); [[fallthrough]];
    case 12: LORPC_TD_PAIR(11); [[fallthrough]];
    case 11: LORPC_TD_PAIR(10); [[fallthrough]];
    case 10: LORPC_TD_PAIR(9); [[fallthrough]];
    case 9: LORPC_TD_PAIR(8); [[fallthrough]];
    case 8: LORPC_TD_PAIR(7); [[fallthrough]];
    case 7: LORPC_TD_PAIR(6); [[fallthrough]];
    case 6: LORPC_TD_PAIR(5); [[fallthrough]];
    case 5: LORPC_TD_PAIR(4); [[fallthrough]];
    case 4: LORPC_TD_PAIR(3); [[fallthrough]];
    case 3: LORPC_TD_PAIR(2); [[fallthrough]];
    case 2: LORPC_TD_PAIR(1); [[fallthrough]];
    case 1: LORPC_TD_PAIR(0); [[fallthrough]];
    default: break;
  }
  return a0 + a1;
}
#undef LORPC_TD_PAIR

// One triangular sweep of the lane's own patch over the T-record block: forward
// (x_i -= sum_{j earlier} L_ij x_j, steps ascending) or backward with the
// diagonal fused (x_i = x_i / D_i - sum_{k later} L_ki x_k, steps descending).
// Software-pipelined one step deep (unrolled by two so that the register stages
// swap roles without moves): the next step's factor rows are loaded while the
// current one is applied, and the record streams through L2 prefetches TPFD pair
// rows ahead.  The kernel instantiates it once (runtime direction, the two
// smoothing steps in a loop), which keeps the kernel inside the instruction cache.
template <int NP>
__device__ __forceinline__ void tsweep(const char* __restrict__ blk, int X, int dummy, bool bwd, int TPFD, int lane) {
  const int4 hd = __ldg((const int4*)blk);
  const int S = hd.x;
  if (S == 0) return;
  const TRecLayout T = trec_layout(S, hd.y, hd.z);
  const int Kp = (bwd ? hd.z : hd.y) / 2, sh = bwd ? 24 : 16, dir = bwd ? -32 : 32;
  const uint32_t* H = (const uint32_t*)(blk + T.hdr) + lane + (bwd ? (S - 1) * 32 : 0);
  const double* Dd = (const double*)(blk + T.D) + lane + (S - 1) * 32;
  const double2* Lp = (const double2*)(blk + (bwd ? T.Lb : T.Lf)) + lane;
  const uint32_t* Cp = (const uint32_t*)(blk + (bwd ? T.Cb : T.Cf)) + lane;
  auto pairs = [&](uint32_t h) { return (int)__reduce_max_sync(0xffffffffu, (((h >> sh) & 0xffu) + 1u) >> 1); };
  // L2 prefetch cursor (pair rows; forward ascending, backward descending)
  int pf = 0;
  auto prefetch = [&](int kp) {
    if (lane != 0) return;
    if (!bwd) {
      while (pf < Kp && pf < kp + TPFD) {
        const int nr = min(8, Kp - pf);
        l2_prefetch(Lp - lane + pf * 32, 512u * nr);
        l2_prefetch(Cp - lane + pf * 32, 128u * nr);
        pf += nr;
      }
    } else {
      while (pf > 0 && pf > kp - TPFD) {
        const int nr = min(8, pf);
        pf -= nr;
        l2_prefetch(Lp - lane + pf * 32, 512u * nr);
        l2_prefetch(Cp - lane + pf * 32, 128u * nr);
      }
    }
  };
  if (lane == 0) {
    l2_prefetch((const uint32_t*)(blk + T.hdr), 128u * S);
    if (bwd) l2_prefetch((const double*)(blk + T.D), 256u * S);
    pf = bwd ? Kp : 0;
  }
  TStage<NP> A, B;
#pragma unroll
  for (int p = 0; p < NP; ++p) A.l[p] = B.l[p] = make_double2(0.0, 0.0);
  uint32_t h0 = __ldg(H), h1 = S > 1 ? __ldg(H + dir) : 0u;
  double d0 = bwd ? __ldg(Dd) : 1.0, d1 = bwd && S > 1 ? __ldg(Dd - 32) : 1.0;
  int m0 = pairs(h0);
  int kp = bwd ? Kp - m0 : 0;  // first pair row of the current step
  prefetch(kp);
  tload<NP>(A, Lp, Cp, kp, m0, (h0 >> sh) & 0xff);
  for (int s = 0; s < S; s += 2) {
    // step s: A current, B <- step s + 1
    const uint32_t h2 = s + 2 < S ? __ldg(H + 2 * dir) : 0u;
    const double d2 = bwd && s + 2 < S ? __ldg(Dd - 64) : 1.0;
    const int m1 = pairs(h1);
    const int kp1 = bwd ? kp - m1 : kp + m0;
    prefetch(kp);
    if (s + 1 < S) tload<NP>(B, Lp, Cp, kp1, m1, (h1 >> sh) & 0xff);
    {
      const int node = h0 & 0xffff;
      double a = tsm[X + node];
      if (bwd) a = a / d0;
      tsm[X + node] = tdot<NP>(A, m0, a, X);
    }
    if (s + 1 >= S) break;
    // step s + 1: B current, A <- step s + 2
    const uint32_t h3 = s + 3 < S ? __ldg(H + 3 * dir) : 0u;
    const double d3 = bwd && s + 3 < S ? __ldg(Dd - 96) : 1.0;
    const int m2 = pairs(h2);
    const int kp2 = bwd ? kp1 - m2 : kp1 + m1;
    if (s + 2 < S) tload<NP>(A, Lp, Cp, kp2, m2, (h2 >> sh) & 0xff);
    {
      const int node = h1 & 0xffff;
      double a = tsm[X + node];
      if (bwd) a = a / d1;
      tsm[X + node] = tdot<NP>(B, m1, a, X);
    }
    H += 2 * dir; Dd -= 64;
    h0 = h2; h1 = h3; d0 = d2; d1 = d3; m0 = m2; kp = kp2;
  }
}

// patch geometry: element box and the free-node boxes of levels 0 and 1
struct TPatch { int lo[3], ext[3], cext[3], ec[3], n, n1; };
static_assert(sizeof(TPatch) % sizeof(double) == 0, "TPatch packs into doubles");
template <int DIM>
__device__ __forceinline__ TPatch tpatch(const PatchGeom& G, long long j) {
  TPatch c;
  int elo[3], ehi[3];
  patch_elems(G, j, elo, ehi);
  c.n = c.n1 = 1;
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    c.ec[k] = ehi[k] - elo[k] + 1;
    if (k >= DIM) { c.lo[k] = 0; c.ext[k] = c.cext[k] = 1; continue; }
    c.lo[k] = elo[k] * (G.ml[0] - 1) + 1;
    c.ext[k] = c.ec[k] * (G.ml[0] - 1) - 1;
    c.cext[k] = c.ec[k] * (G.ml[1] - 1) - 1;
    c.n *= c.ext[k];
    c.n1 *= c.cext[k];
  }
  return c;
}

// ------------------------------------------------------------------ middle phase
// Lane = patch, no shared memory (high occupancy); the patch vectors are the
// lane's columns of warp-interleaved global buffers [warp][node][32] (every access
// of a warp is one 256-byte row).  x: pre-smoothed iterate, y: after the coarse
// correction, s: residual handed to the post-smoothing.

// Thread mode: coarse-level box bound per axis (tmode requires n_1 <= 32)
template <int DIM> struct TCoarse {
  static constexpr int CX = DIM == 3 ? 3 : 5, CZ = DIM == 3 ? 3 : 1, NC = CX * CX * CZ;
};

// 1D restriction weights of fine node (ix, iy, iz) to the coarse box (dense W[c][f],
// zero off the hat support)
template <int DIM>
__device__ __forceinline__ void tweights(const TcParams& P, const TPatch& c, int ix, int iy, int iz, double* wx,
                                         double* wy, double* wz) {
  constexpr int CX = TCoarse<DIM>::CX, CZ = TCoarse<DIM>::CZ;
  const double* Wx = P.W + P.woff[c.ec[0]];
  const double* Wy = P.W + P.woff[c.ec[1]];
  const double* Wz = P.W + P.woff[DIM == 3 ? c.ec[2] : 1];
#pragma unroll
  for (int k = 0; k < CX; ++k) {
    wx[k] = k < c.cext[0] ? __ldg(Wx + k * c.ext[0] + ix) : 0.0;
    wy[k] = k < c.cext[1] ? __ldg(Wy + k * c.ext[1] + iy) : 0.0;
  }
#pragma unroll
  for (int k = 0; k < CZ; ++k) wz[k] = DIM == 3 ? (k < c.cext[2] ? __ldg(Wz + k * c.ext[2] + iz) : 0.0) : 1.0;
}

// s_i = r_i - (A_0 v)_i at node i of the lane's patch, v = the lane's column V
template <int DIM>
__device__ __forceinline__ double tres_node(const TcParams& P, const TPatch& c, const double* __restrict__ V, int i,
                                            int ix, int iy, int iz) {
  constexpr int ND = Dirs<DIM>::ND, NDP = Dirs<DIM>::NDP;
  const int ex = c.ext[0], ey = c.ext[1], ez = c.ext[2];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  const unsigned gi = (unsigned)((c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (DIM == 3 ? c.lo[2] + iz : 0)));
  const uint32_t em = exist_mask<DIM>(ix, iy, iz, ex, ey, ez);
  double a0 = __ldg(P.r + gi), a1 = 0.0;
  const double2* Ar = (const double2*)(P.A0 + (size_t)gi * NDP);
#pragma unroll
  for (int d2 = 0; d2 < NDP / 2; ++d2) {
    const double2 av = __ldg(Ar + d2);
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int d = 2 * d2 + h;
      if (d >= ND) break;
      const int o = dir_dx(d) + ex * (dir_dy(d) + ey * (DIM == 3 ? dir_dz(d) : 0));
      const double v = (em & (1u << d)) ? V[(i + o) * 32] : 0.0;
      if (h) a1 -= av.y * v; else a0 -= av.x * v;
    }
  }
  return a0 + a1;
}

template <int DIM>
__global__ void __launch_bounds__(128) k_vt_mid(TcParams P) {
  constexpr int CX = TCoarse<DIM>::CX, CZ = TCoarse<DIM>::CZ, NC = TCoarse<DIM>::NC, NC1 = 32;
  const long long j = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long w = j >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= P.J) return;
  const TPatch c = tpatch<DIM>(P.G, j);
  const int n0 = P.n0max, ex = c.ext[0], ey = c.ext[1];
  const float rex = 1.0f / ex, rexy = 1.0f / (ex * ey);
  const long long col = w * (long long)n0 * 32 + lane;
  const double* Xp = P.xpark + col;
  double* Yp = P.ypark + col;
  double* Sp = P.spark + col;
  // s = r - A x and r_1 = P^T s (fused)
  double r1[NC];
#pragma unroll
  for (int k = 0; k < NC; ++k) r1[k] = 0.0;
  for (int f = 0; f < c.n; ++f) {
    int ix, iy, iz;
    box_xyz(f, ex, ey, rex, rexy, ix, iy, iz);
    const double sv = tres_node<DIM>(P, c, Xp, f, ix, iy, iz);
    double wx[CX], wy[CX], wz[CZ];
    tweights<DIM>(P, c, ix, iy, iz, wx, wy, wz);
#pragma unroll
    for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
      for (int ky = 0; ky < CX; ++ky) {
        const double wv = wy[ky] * wz[kz] * sv;
#pragma unroll
        for (int kx = 0; kx < CX; ++kx) r1[kx + CX * (ky + CX * kz)] += wx[kx] * wv;
      }
  }
  // z_1 = C r_1: r_1 to the patch's coarse numbering, C interleaved by lane
  const int n1 = c.n1, cx = c.cext[0], cy = c.cext[1], cz = c.cext[2];
  double* R = P.rz + w * 2ll * P.n1max * 32 + lane;
  double* Z = R + P.n1max * 32;
#pragma unroll
  for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
    for (int ky = 0; ky < CX; ++ky)
#pragma unroll
      for (int kx = 0; kx < CX; ++kx)
        if (kx < cx && ky < cy && kz < cz) R[(kx + cx * (ky + cy * kz)) * 32] = r1[kx + CX * (ky + CX * kz)];
  {
    const double* C = P.Cd + w * 32ll * P.ldc + lane;
    double zc[NC1];
#pragma unroll
    for (int i = 0; i < NC1; ++i) zc[i] = 0.0;
    for (int k = 0; k < n1; ++k) {
      const double rk = R[k * 32];
      const double* Ck = C + (long long)k * n1 * 32;
#pragma unroll
      for (int i = 0; i < NC1; ++i)
        if (i < n1) zc[i] += __ldcs(Ck + i * 32) * rk;
    }
#pragma unroll
    for (int i = 0; i < NC1; ++i)
      if (i < n1) Z[i * 32] = zc[i];
  }
  // y = x + P z_1
  double z1[NC];
#pragma unroll
  for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
    for (int ky = 0; ky < CX; ++ky)
#pragma unroll
      for (int kx = 0; kx < CX; ++kx)
        z1[kx + CX * (ky + CX * kz)] = (kx < cx && ky < cy && kz < cz) ? Z[(kx + cx * (ky + cy * kz)) * 32] : 0.0;
  for (int f = 0; f < c.n; ++f) {
    int ix, iy, iz;
    box_xyz(f, ex, ey, rex, rexy, ix, iy, iz);
    double wx[CX], wy[CX], wz[CZ];
    tweights<DIM>(P, c, ix, iy, iz, wx, wy, wz);
    double t = 0.0;
#pragma unroll
    for (int kz = 0; kz < CZ; ++kz)
#pragma unroll
      for (int ky = 0; ky < CX; ++ky) {
        double u = 0.0;
#pragma unroll
        for (int kx = 0; kx < CX; ++kx) u += wx[kx] * z1[kx + CX * (ky + CX * kz)];
        t += wy[ky] * wz[kz] * u;
      }
    Yp[f * 32] = Xp[f * 32] + t;
  }
  // s = r - A y
  for (int f = 0; f < c.n; ++f) {
    int ix, iy, iz;
    box_xyz(f, ex, ey, rex, rexy, ix, iy, iz);
    __stcs(Sp + f * 32, tres_node<DIM>(P, c, Yp, f, ix, iy, iz));
  }
}

// ------------------------------------------------------------------ smoothing phases
// pre (POST = false): X = r_j (gather), X = M^{-1} X, x -> xpark.
// post (POST = true): X = s (spark), X = M^{-1} X, z += I_j (y + X) (a8).
template <int DIM, bool POST>
__global__ void __launch_bounds__(32) k_vt_smooth(TcParams P) {
  constexpr int NP = DIM == 3 ? 13 : 4;
  const int lane = threadIdx.x;
  const long long w = blockIdx.x;
  const int X = 0, n0 = P.n0max;
  const int nq = (int)min(32ll, P.J - w * 32);
  const char* blk = P.trec + P.trecoff[w];
  const long long Nx = P.G.Nax[0][0], Ny = P.G.Nax[0][1];
  TPatch* tpa = (TPatch*)(tsm + P.tpoff);
  if (lane < nq) tpa[lane] = tpatch<DIM>(P.G, w * 32 + lane);
  const long long col = w * (long long)n0 * 32 + lane;
  if (!POST) {
    __syncwarp();
    for (int q = 0; q < nq; ++q) {  // r_j = I_j^T r (a5)
      const TPatch c = tpa[q];
      const float rex = 1.0f / c.ext[0], rexy = 1.0f / (c.ext[0] * c.ext[1]);
      for (int i = lane; i < c.n; i += 32) {
        int ix, iy, iz;
        box_xyz(i, c.ext[0], c.ext[1], rex, rexy, ix, iy, iz);
        tsm[X + VO(i, q)] = __ldg(P.r + (c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (DIM == 3 ? c.lo[2] + iz : 0)));
      }
    }
  } else {
    for (int i = 0; i < n0; ++i) tsm[X + VO(i, lane)] = __ldcs(P.spark + col + i * 32);
  }
  tsm[X + VO(n0, lane)] = 0.0;  // dummy node of the padded sweep steps
  __syncwarp();
#pragma unroll 1
  for (int sw = 0; sw < 2; ++sw) tsweep<NP>(blk, X, n0, sw == 1, P.pfd, lane);
  if (!POST) {
    for (int i = 0; i < n0; ++i) __stcs(P.xpark + col + i * 32, tsm[X + VO(i, lane)]);
  } else {
    for (int i = 0; i < n0; ++i) tsm[X + VO(i, lane)] += __ldcs(P.ypark + col + i * 32);
    __syncwarp();
    for (int q = 0; q < nq; ++q) {  // z += I_j z_j (a8), lanes over consecutive nodes
      const TPatch c = tpa[q];
      const float rex = 1.0f / c.ext[0], rexy = 1.0f / (c.ext[0] * c.ext[1]);
      for (int i = lane; i < c.n; i += 32) {
        int ix, iy, iz;
        box_xyz(i, c.ext[0], c.ext[1], rex, rexy, ix, iy, iz);
        atomicAdd(P.z + (c.lo[0] + ix) + Nx * ((c.lo[1] + iy) + Ny * (DIM == 3 ? c.lo[2] + iz : 0)),
                  tsm[X + VO(i, q)]);
      }
    }
  }
}

static TcParams make_tparams(const lorpc_prec* b, const double* r, double* z) {
  TcParams P{};
  P.G = make_geom(b);
  P.A0 = b->lor->A[0];
  P.W = b->wtab;
  memcpy(P.woff, b->woff[0], sizeof(P.woff));
  P.trec = b->trec; P.trecoff = b->trecoff; P.J = b->J;
  P.Cd = b->Cdi; P.ldc = b->ldc;
  P.n0max = b->max_n[0]; P.n1max = b->max_n[1];
  const long long nw = (b->J + 31) / 32, pcol = nw * b->max_n[0] * 32;
  P.xpark = b->zpark; P.ypark = b->zpark + pcol; P.spark = b->zpark + 2 * pcol; P.rz = b->zpark + 3 * pcol;
  P.r = r; P.z = z;
  int acc = VO(b->max_n[0] + 1, 0);
  P.tpoff = acc; acc += 32 * (int)(sizeof(TPatch) / sizeof(double));
  P.warp_doubles = (acc + 1) & ~1;
  P.pfd = getenv("LORPC_TPFD") ? atoi(getenv("LORPC_TPFD")) : 32;
  return P;
}

size_t tmode_smem(const lorpc_prec* b) {
  return (size_t)make_tparams(b, nullptr, nullptr).warp_doubles * sizeof(double);
}

int vcycle_t_apply(const lorpc_prec* b, const double* r, double* z, cudaStream_t s) {
  const TcParams P = make_tparams(b, r, z);
  const size_t smem = (size_t)P.warp_doubles * sizeof(double);
  if (smem > 227 * 1024) return fail(LORPC_ERR_SIZE, "vcycle_t: warp vectors do not fit in shared memory");
  const unsigned wblocks = (unsigned)((b->J + 31) / 32), mblocks = (unsigned)((b->J + 127) / 128);
  if (b->m->d == 2) {
    cudaFuncSetAttribute(k_vt_smooth<2, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_vt_smooth<2, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_vt_smooth<2, false><<<wblocks, 32, smem, s>>>(P);
    LORPC_LAUNCHED();
    k_vt_mid<2><<<mblocks, 128, 0, s>>>(P);
    LORPC_LAUNCHED();
    k_vt_smooth<2, true><<<wblocks, 32, smem, s>>>(P);
  } else {
    cudaFuncSetAttribute(k_vt_smooth<3, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    cudaFuncSetAttribute(k_vt_smooth<3, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    k_vt_smooth<3, false><<<wblocks, 32, smem, s>>>(P);
    LORPC_LAUNCHED();
    k_vt_mid<3><<<mblocks, 128, 0, s>>>(P);
    LORPC_LAUNCHED();
    k_vt_smooth<3, true><<<wblocks, 32, smem, s>>>(P);
  }
  LORPC_LAUNCHED();
  return LORPC_OK;
}

}  // namespace lorpc
