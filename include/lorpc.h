/*
 * lorpc.h — C ABI of the B200-native LOR additive-Schwarz preconditioned PCG
 * hot path of arXiv 1908.07071 ("Matrix-free preconditioners for high-order
 * continuous and discontinuous Galerkin discretizations").
 *
 * Citations: "P:n" = PAPER.md line n (section / \label named); readings "cN"
 * are listed in DESIGN.md §Readings.
 *
 * Conventions (all entry points):
 *  - Return value: LORPC_OK (0) or an lorpc_status error code.  No exceptions
 *    or exit() cross the ABI; a human-readable diagnostic of the last error on
 *    the calling thread is available from lorpc_last_error().
 *  - Pointers ending in `_dev` are CUDA device pointers (FP64 unless stated),
 *    owned by the caller, which must keep them alive until the stream work that
 *    uses them has completed.  `_host` pointers are host memory.
 *  - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *    All apply calls are asynchronous on that stream; setup calls and
 *    lorpc_pcg_solve synchronize the stream before returning.
 *  - Handles (lorpc_mesh, lorpc_lor, lorpc_prec) own their device workspaces,
 *    allocated at create/setup time and never inside apply/solve; destroy frees
 *    them.  A lorpc_lor / lorpc_prec references its mesh, which must outlive it.
 *  - Layout: CG vectors have one entry per GLL node of the global node grid
 *    (n_0 p + 1) x (n_1 p + 1) [x (n_2 p + 1)], x fastest, Dirichlet (grid
 *    boundary) entries present.  DG vectors are element-major
 *    [n_el][(p+1)^d], elements x-fastest, local nodes x-fastest.
 *  - Mesh: Cartesian topology n_0 x n_1 [x n_2] of tensor-product elements, each
 *    the image of [0,1]^d under the multilinear map of its 2^d vertices
 *    (P:82-84); vertices [(n_0+1)(n_1+1)[(n_2+1)]][d], x fastest.
 */
#ifndef LORPC_H
#define LORPC_H

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  LORPC_OK = 0,
  LORPC_ERR_ARG = 1,              /* invalid argument (NULL, p < 1, eta <= 0, ...) */
  LORPC_ERR_SIZE = 2,             /* unsupported size (p outside the compiled set, ...) */
  LORPC_ERR_INVERTED_ELEMENT = 3, /* det J <= 0 at a quadrature point (element id in message) */
  LORPC_ERR_ZERO_PIVOT = 4,       /* ILU(0) pivot <= 0 (patch, level, step in message) */
  LORPC_ERR_BREAKDOWN = 5,        /* PCG p.Ap <= 0 or r.z <= 0 (iteration in message) */
  LORPC_ERR_NOT_CONVERGED = 6,    /* PCG hit maxit */
  LORPC_ERR_CUDA = 7,             /* CUDA runtime error */
  LORPC_ERR_OOM = 8,              /* device allocation failed */
  LORPC_ERR_NOT_SPD = 9,          /* a matrix that must be SPD is not (coarsest R_0 level: Cholesky pivot <= 0) */
  LORPC_ERR_NCCL = 10             /* NCCL error in the multi-GPU path (lorpc_dist_*) */
} lorpc_status;

typedef struct lorpc_mesh lorpc_mesh;
typedef struct lorpc_lor lorpc_lor;
typedef struct lorpc_prec lorpc_prec;

/* Discretisation (P:82-105 CG, eq:ip P:113-136 SIPG). */
typedef struct {
  int dim;      /* 2 or 3 */
  int n[3];     /* elements per axis (n[2] ignored in 2D) */
  int p;        /* polynomial degree; compiled set: 2D p in {2..8}, 3D p in {2..6} */
  int disc;     /* 0 = continuous H1 (CG), 1 = symmetric interior penalty DG (eq:ip),
                   2 = BR2 DG (eq:br2 P:152-158, lifting eq:lift P:662-665; affine elements only,
                   LORPC_ERR_SIZE otherwise).  DG requires dim = 3. */
  double eta;   /* SIPG: sigma_e = eta / h_e, h_e = min(|K-|,|K+|)/|e| (readings c13, c14);
                   BR2: coefficient of sum_e (r_e([u]), r_e([v])) */
  int quad;     /* volume quadrature: 0 = Gauss q = p+1 (reading c1), 1 = GLL collocation
                   (the p+1 GLL nodes per direction; SURVEY row f2, P:785-793 quadrature
                   variant).  quad = 1 requires disc = 0 (LORPC_ERR_ARG otherwise). */
} lorpc_mesh_desc;

/* Additive Schwarz B = sum_{j=0}^J R_j Q_j (eq:as P:274-277). */
typedef struct {
  int patch_kind; /* 0 = vertex patches (eq:patch P:302-315), 1 = element star (reading c9),
                     2 = single patch B(1): one element-structured V-cycle on the whole
                     LOR problem with R_0 at its p = 1 bottom (requires coarse = 0; levels of at
                     most 65535 free nodes) */
  int ordering;   /* ILU(0) ordering: 0 = minimum discarded fill, 1 = natural,
                     2 = reverse Cuthill-McKee (structure only, reading r5) */
  int coarse;     /* 0 = R_0 one GMG V(1,1) with l1-Jacobi (reading c11), 1 = no coarse term */
  int extend;     /* 1 = vertex patches extended for isotropic overlap (sec:aniso P:1123-1128,
                     rem:anisotropy P:499-502; rule: reading r6, single rank, vertex patches
                     only); 0 = eq:patch as is */
} lorpc_schwarz_desc;

typedef struct {
  int iters;          /* operator applications performed */
  int converged;      /* 1 if ||r||_2 <= rtol ||b||_2 */
  double rel_res;     /* final ||r||_2 / ||b||_2 (recursively updated residual) */
  double* res_hist;   /* host, caller-owned, length >= maxit+1, or NULL */
  double* alpha;      /* host, length >= maxit, or NULL (Lanczos kappa) */
  double* beta;       /* host, length >= maxit, or NULL */
  double t_solve_ms;  /* device time of the iteration loop (CUDA events) */
} lorpc_pcg_report;

/* ---- mesh / geometry (a1) ------------------------------------------------- */
/* Creates the mesh, uploads the vertices, computes geometric factors
 * G_q = w_q det J_q J_q^{-1} J_q^{-T} at the q^d Gauss points (q = p+1,
 * reading c1) and checks det J > 0 (LORPC_ERR_INVERTED_ELEMENT). */
int lorpc_mesh_create(const lorpc_mesh_desc* desc, const double* vertices_host, void* stream,
                      lorpc_mesh** out);
void lorpc_mesh_destroy(lorpc_mesh* m);
/* Sizes: n_dof = length of the solution vector (CG nodes or DG dofs), n_quad =
 * number of volume quadrature points, n_bface_quad = boundary-face quadrature
 * points (DG weak Dirichlet data, reading c15; 0 for CG). */
int lorpc_mesh_sizes(const lorpc_mesh* m, long long* n_dof, long long* n_quad, long long* n_bface_quad);
/* Physical coordinates [n_quad][d] of the volume Gauss points (element-major,
 * x-fastest) and [n_bface_quad][d] of the boundary-face Gauss points (ordering:
 * axis, side low/high, elements ascending, face points lower axis fastest);
 * either output may be NULL. */
int lorpc_quad_points(const lorpc_mesh* m, double* xq_dev, double* xbq_dev, void* stream);
/* Variable coefficient b(x) of -div(b grad u) (row f3; P:881-901,
 * sec:variable-coeff, coefficients b1..b4 there).  bq_dev [n_quad] = b at the
 * volume Gauss points in the lorpc_quad_points order (enters K_p as b(x_q) w_q
 * det J J^{-1} J^{-T}); bsub_dev [n_sub * 2^d] = b at the Gauss points of the LOR
 * subcells in the lorpc_subcell_points order (enters K_h, sampled pointwise: SPEC
 * S:233 reading).  Either may be NULL (b = 1).  Device arrays, copied; the mesh's
 * geometric factors are re-formed.  Must precede lorpc_lor_assemble.  CG meshes
 * only.  Errors: LORPC_ERR_ARG (DG mesh, a value <= 0). */
int lorpc_mesh_set_coefficient(lorpc_mesh* m, const double* bq_dev, const double* bsub_dev, void* stream);
/* Gauss points of the LOR subcells (2^d per subcell, t = 1/2 -+ 1/(2 sqrt 3) on the
 * subcell map multilinear in its corner GLL node images, reading c2): xs_dev
 * [n_sub][2^d][d], subcell index sx + (N0-1)(sy + (N1-1) sz) major (N = GLL nodes per
 * axis), Gauss-point bits x, y, z minor; *n_sub = number of subcells.  xs_dev may be
 * NULL (size query only). */
int lorpc_subcell_points(const lorpc_mesh* m, double* xs_dev, long long* n_sub, void* stream);
/* Load vector b = (f, v) (eq:fem) from f at the volume Gauss points; CG:
 * Dirichlet rows zeroed; DG: plus the symmetric Nitsche boundary data
 * int_e (sigma_e g v - g d_n v) from g at the boundary points (gq_dev may be
 * NULL for g = 0). */
int lorpc_rhs_assemble(const lorpc_mesh* m, const double* fq_dev, const double* gq_dev,
                       double* b_dev, void* stream);

/* ---- operator (a2, a3) ------------------------------------------------------ */
/* y = A x, matrix-free by sum factorisation (tab:complexity P:764).
 * CG: y_F = K_FF x_F, y_D = x_D (symmetric Dirichlet elimination).
 * SIPG: volume term plus interior/boundary face terms of eq:ip.
 * x_dev and y_dev must not alias. */
int lorpc_operator_apply(const lorpc_mesh* m, const double* x_dev, double* y_dev, void* stream);

/* ---- LOR (a11) ---------------------------------------------------------------- */
/* Assembles K_h, the Q1 stiffness on the GLL-refined mesh (exact
 * multilinear subcell maps with 2^d Gauss points, reading c2), and the
 * element-structured Galerkin hierarchy A_{l+1} = P_l^T A_l P_l (P:549-555,
 * readings c3, c4).  For a DG mesh the CG LOR of the same mesh and p is built
 * (R_p of eq:dg-as). */
int lorpc_lor_assemble(const lorpc_mesh* m, void* stream, lorpc_lor** out);
void lorpc_lor_destroy(lorpc_lor* l);

/* ---- Schwarz setup (a5-a9, a11) ------------------------------------------------ */
/* Patches, per-patch per-level ordering (MDF, reading c6) fused with the ILU(0)
 * elimination into M = L D L^T (reading c5), level schedules, the coarse-space
 * GMG hierarchy (reading c11) and, for DG, D_B = diag(A_IP) on element-boundary
 * DG nodes (reading c16).  Errors: LORPC_ERR_ZERO_PIVOT. */
int lorpc_schwarz_setup(const lorpc_lor* l, const lorpc_schwarz_desc* desc, void* stream,
                        lorpc_prec** out);
void lorpc_prec_destroy(lorpc_prec* b);
/* z = B r (eq:as); CG: z_D = 0.  DG: z = E B(E^T r) + S_B D_B^{-1} S_B^T r
 * (eq:dg-as P:635-641).  r_dev and z_dev must not alias. */
int lorpc_precond_apply(const lorpc_prec* b, const double* r_dev, double* z_dev, void* stream);
/* Copies the elimination order (patch-local natural indices, step order) of
 * patch `patch` at hierarchy level `level` to perm_host (capacity *n on input;
 * the patch size on output). */
int lorpc_prec_export_ordering(const lorpc_prec* b, long long patch, int level, int* perm_host, int* n);
/* Number of patches and hierarchy levels. */
int lorpc_prec_info(const lorpc_prec* b, long long* n_patches, int* n_levels);
/* Which patch V-cycle kernel family lorpc_precond_apply runs (a5-a8; for bench
 * labels): 0 = group mode (k_vcycle: VG lanes per patch, every level in shared
 * memory), 1 = thread mode (vcycle_t.cu: one lane per patch, warp-interleaved
 * factors), 2 = W mode (vcycle_w.cu: warp-per-patch fused V-cycle, opt-in through
 * LORPC_WMODE=1), 3 = thread mode with U-records (structure-only orderings: natural,
 * RCM; the warp's patches share one sweep schedule, only factor values per lane),
 * 4 = Q mode (vcycle_w.cu: fused V-cycle with 2 / 4 / 8 lanes per patch, one sweep
 * schedule per warp, factors streamed through a cp.async ring; LORPC_QMODE=1).
 * Errors: LORPC_ERR_ARG on NULL. */
int lorpc_prec_kernel(const lorpc_prec* b, int* mode);
/* Algorithmic byte-model inputs: factor_values = sum over
 * patches and levels of (free nodes + stencil edges), i.e. the L and D values of
 * every M_l = L D L^T; level_nodes[l] = nodes of the level-l grid (l < n_levels),
 * coarse_nodes = nodes of all R_0 GMG levels. */
int lorpc_prec_bytes(const lorpc_prec* b, long long* factor_values, long long* level_nodes, long long* coarse_nodes);
/* Live timing of the patch V-cycle kernel (the dominant kernel): enable = 1
 * starts recording a CUDA event pair around every launch on the apply stream
 * (up to 4096 launches), enable = 0 stops; lorpc_prec_profile_read synchronizes
 * and returns the summed device time (ms) and launch count, then resets. */
int lorpc_prec_profile(lorpc_prec* b, int enable);
int lorpc_prec_profile_read(lorpc_prec* b, double* ms, long long* launches);

/* ---- PCG (a10) ------------------------------------------------------------------ */
/* Preconditioned conjugate gradients (reading c12): x_0 = 0,
 * stop when ||r_k||_2 <= rtol ||b||_2.  CG: b's Dirichlet entries must be zero
 * (homogeneous Dirichlet, as lorpc_rhs_assemble writes them; B has zero rows there,
 * so a nonzero b_D cannot be reduced and the solve ends in NOT_CONVERGED or
 * BREAKDOWN).  x_dev is overwritten.  Device-resident
 * vectors; synchronizes the stream.  Returns LORPC_ERR_NOT_CONVERGED or
 * LORPC_ERR_BREAKDOWN with the report filled up to the last iteration. */
int lorpc_pcg_solve(const lorpc_mesh* m, const lorpc_prec* b, const double* b_dev, double* x_dev,
                    double rtol, int maxit, lorpc_pcg_report* rep, void* stream);
/* Same solve with host buffers: copies b_host in and x_host out inside the
 * call (the end-to-end path the bench's e2e number times). */
int lorpc_pcg_solve_host(const lorpc_mesh* m, const lorpc_prec* b, const double* b_host, double* x_host,
                         double rtol, int maxit, lorpc_pcg_report* rep, void* stream);

/* ---- multi-GPU slab decomposition (BASELINE C5 "element slabs
 * partitioned across 1/2/4/8 GPUs with NCCL halo exchange") ------------------ */
/* 3D CG only.  Rank r of R owns element layers [z0, z1) along z (balanced:
 * z0 = floor(n_z r / R)), node planes [z0 p, z1 p) and vertex planes [z0, z1)
 * (the last rank also the top plane): its owned nodes are one contiguous range
 * of the global node vector (z is the slowest axis).  It builds a local sub-mesh
 * of element layers [za, zb) = [z0 - 1, z1 + 1] clipped to the domain from the
 * replicated vertex array (one ghost layer per side), so LOR rows, patch factors
 * (vertex patches of its owned vertex planes, eq:patch P:302-315) and coarse rows
 * are computed locally; R_0 (reading c11) runs replicated on the gathered global
 * vertex-level operator.  Per PCG iteration four point-to-point exchanges
 * (phases below), one allreduce of the coarse residual on the vertex grid and
 * the scalar allreduces. */
typedef struct {
  int z0, z1, za, zb;          /* owned / local element layers (global indices) */
  int own_plane0, own_planes;  /* owned node planes: local index of the first, count */
  int gown_plane0;             /* global index of the first owned node plane */
  int vown0, nvown;            /* owned vertex planes: local index of the first, count */
  /* phase k: 0 = operator input (copy), 1 = operator output partial sums (add on
   * free nodes), 2 = Schwarz input r halo (copy), 3 = Schwarz output patch sums
   * (add).  Send nplanes[k] planes from local plane send0[k] to rank to[k];
   * receive nplanes[k] planes into local plane recv0[k] from rank from[k]; -1 =
   * none. */
  int to[4], from[4], send0[4], recv0[4], nplanes[4];
} lorpc_dist_plan;
typedef struct lorpc_dist lorpc_dist;
/* The slab plan of rank `rank` (host only, no device work): LORPC_ERR_ARG unless
 * n_z >= nranks >= 1 and p >= 1. */
int lorpc_dist_plan_get(int n_z, int p, int nranks, int rank, lorpc_dist_plan* out);
/* ncclGetUniqueId (128 bytes) — called on rank 0, broadcast by the caller. */
int lorpc_dist_nccl_id(void* id128);
/* Builds the rank's local problem.  desc / vertices_host describe the GLOBAL
 * mesh.  nccl_id != NULL: one rank per process (device = current device),
 * NCCL communicator of nranks ranks (collective call).  nccl_id == NULL:
 * emulation — all nranks ranks in this process on the current device, the
 * exchanges done by device copies (testing the multi-rank path on one GPU).
 * sdesc must request vertex patches with the GMG coarse term.  Synchronizes. */
int lorpc_dist_create(const lorpc_mesh_desc* desc, const double* vertices_host, const lorpc_schwarz_desc* sdesc,
                      int nranks, int rank, const void* nccl_id, void* stream, lorpc_dist** out);
void lorpc_dist_destroy(lorpc_dist* d);
/* Local rank `local` (0 in NCCL mode; 0..nranks-1 in emulation): global index of
 * its first owned node, owned node count, patch count. */
int lorpc_dist_info(const lorpc_dist* d, int local, long long* owned_offset, long long* n_owned, long long* n_patches);
/* The rank's local patch preconditioner (owned vertex-plane patches, no coarse
 * term; owned by d): for lorpc_prec_info / lorpc_prec_bytes (byte model). */
int lorpc_dist_local_prec(const lorpc_dist* d, int local, const lorpc_prec** out);
/* y = A x and z = B r on the distributed vectors: arrays of one device pointer per
 * local rank, each the rank's owned range [owned_offset, owned_offset + n_owned)
 * of the global vector.  Asynchronous on the creation stream. */
int lorpc_dist_operator_apply(lorpc_dist* d, const double* const* x_owned, double* const* y_owned);
int lorpc_dist_precond_apply(lorpc_dist* d, const double* const* r_owned, double* const* z_owned);
/* PCG (as lorpc_pcg_solve) on the distributed vectors; dot products are global
 * (fixed order per rank, then summed over ranks).  Synchronizes. */
int lorpc_dist_pcg_solve(lorpc_dist* d, const double* const* b_owned, double* const* x_owned, double rtol,
                         int maxit, lorpc_pcg_report* rep);

/* Number of kernel launches issued by this library on the calling thread since
 * the last reset (instrumentation for the bench's gpu_launches claim). */
long long lorpc_launch_count(int reset);
const char* lorpc_last_error(void);

#ifdef __cplusplus
}
#endif
#endif /* LORPC_H */
