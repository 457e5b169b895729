/*
 * dot_b200.h -- C ABI of the B200-native DOT hot path (arXiv 1706.05586).
 *
 * The library (paper_1706_05586_b200/lib/libdot_b200.so) solves the batched
 * multi-right-hand-side frequency-domain diffusion systems of PAPER.md Eq. (2.1)
 * and evaluates the sketched misfit, the co-state Jacobian and the simultaneous
 * optimized sources/detectors of Sec. 3 -- all steps in hand-written sm_100a
 * CUDA kernels.  No torch types cross this boundary: plain pointers and sizes.
 *
 * Conventions (all calls)
 *   - Return value: DOT_OK (0) or a DOT_ERR_* code; dot_last_error() gives text.
 *     No call aborts the process.  On error the output buffers are unspecified.
 *   - `where` = DOT_HOST or DOT_DEVICE says where ALL array arguments of that
 *     call live (scalars returned through `double* ..._out` marked "(host)" are
 *     always host).  Device pointers must be 16-byte aligned and belong to the
 *     device the problem was created on.  Host pointers may be pageable; pinned
 *     host memory gives asynchronous copies.
 *   - Complex numbers are interleaved (re, im) doubles.  All arithmetic is
 *     complex fp64 / fp64.
 *   - Ownership: the caller owns every buffer it passes; the library never
 *     frees them.  Device memory used by the library comes from ONE workspace
 *     the caller binds with dot_bind_workspace (e.g. a torch uint8 tensor).
 *   - Ordering: every call enqueues on the stream set by dot_set_stream (default
 *     stream if unset) and returns after its results are complete on that
 *     stream for host outputs; device outputs are complete in stream order.
 *
 * Grid (readings R1-R3): interior FD nodes of [0,Lx]x[0,Ly]x[0,Lz]:
 *   x_i = (i+1) Lx/(nx+1), y_j = (j+1) Ly/(ny+1)  (phi = 0 on the lateral faces,
 *   PAPER.md L136), z_k = k Lz/(nz-1) including the Robin planes z = 0 and
 *   z = Lz (L137).  Node (i,j,k) has linear index n = (k*ny + j)*nx + i.
 *   Fields are [N] complex arrays in that order, N = nx*ny*nz.
 */
#ifndef DOT_B200_H
#define DOT_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DOT_OK 0
#define DOT_ERR_ARG 1        /* invalid argument / size / pointer            */
#define DOT_ERR_CUDA 2       /* CUDA runtime error (text in dot_last_error)  */
#define DOT_ERR_STATE 3      /* call order (e.g. misfit before set_params)   */
#define DOT_ERR_NOCONV 4     /* a Krylov solve hit max_iter                  */
#define DOT_ERR_WORKSPACE 5  /* bound workspace too small for the request    */
#define DOT_ERR_BREAKDOWN 6  /* CG breakdown (p^T K p <= 0 or non-finite)     */

#define DOT_HOST 0
#define DOT_DEVICE 1

typedef struct dot_problem dot_problem;
typedef struct dot_dd dot_dd;          /* z-slab domain-decomposition group */

/* Problem description.  All pointers are HOST pointers, copied by dot_create. */
typedef struct dot_config {
    int32_t nx, ny, nz;          /* interior nodes; nx,ny >= 1, nz >= 2, nx <= 256        */
    double Lx, Ly, Lz;           /* domain extents (cm)                                   */
    double D;                    /* diffusion coefficient (cm), constant (reading R4)     */
    double mua_in, mua_out;      /* absorption inside / outside the level set (1/cm), Eq. (2.4) */
    double nu;                   /* speed of light in the medium (cm/s), Eq. (2.1)        */
    int32_t n_freq;              /* number of modulation frequencies                      */
    const double* omega;         /* [n_freq] angular frequencies omega (rad/s)            */
    int32_t n_src;               /* point sources b_s = theta e_node / (hx hy hz) (reading R6) */
    const int64_t* src_nodes;    /* [n_src] linear node indices                           */
    int32_t n_det;               /* point detectors c_d = e_node                          */
    const int64_t* det_nodes;    /* [n_det] linear node indices                           */
    int32_t n_rbf;               /* PaLS basis functions; n_p = 5 n_rbf (Eq. (2.3))      */
    double gamma;                /* ||x||^dagger regulariser              */
    double eps;                  /* smoothed-Heaviside half width (reading R8)            */
    double cutoff;               /* level-set cut-off c (Eq. (2.4))                       */
    double tol;                  /* Krylov stop per system: ||r_sigma||_2 <= tol ||b||_2 (reading R12); <=0: 1e-17 */
    int32_t max_iter;            /* Krylov iteration cap; <= 0: 4000                      */
} dot_config;

typedef struct dot_stats {
    int64_t rhs_solved;          /* PDE systems A(p, omega_f) x = b solved since create, one per
                                    (right-hand side, frequency) (Table 4 accounting) */
    int64_t rhs_iterations;      /* sum over solved systems of the Krylov iterations they took */
    int32_t last_max_iters;      /* max iterations of the last batched solve              */
    int32_t last_min_iters;
    int64_t kernel_launches;     /* kernels launched by the library since create          */
    int64_t pass_launches;       /* fused CG pass launches since create                   */
    double pass_ms;              /* device time in CG pass kernels (when timing enabled)  */
    double pass_bytes;           /* algorithmic HBM bytes of those passes: 32 B x N per real seed
                                    per iteration (read r, p; write r, p in fp64)            */
    double contract_ms;          /* device time in the Jacobian contraction (timing enabled) */
    double contract_flops;       /* its useful flops: 4 x pairs x (points, parameter) pairs with a
                                    nonzero dA/dp block (block-sparse by basis, L972)            */
    int32_t support_K;           /* |S|: nodes where dA/dp != 0 after the last set_params */
    int32_t n_samples;           /* |P| = |S u detectors u sources|: nodes where solutions are kept */
    double contract_flops_dense; /* the dense-equivalent flops 4 x pairs x K x n_p of the same calls */
    int64_t seeds_solved;        /* real multi-shift CG seeds run (one serves every frequency)   */
    int64_t seed_iterations;     /* sum over seeds of their iterations                           */
    double contract_dmma_flops;  /* FP64 tensor (DMMA) flops the segment GEMM executed: 3 real
                                    products per complex one, padded tiles included (the useful
                                    flops above are 2/3 of it at most)                           */
    double gemm_ms;              /* the part of contract_ms spent in calls that took the segment
                                    GEMM path (large panels: the full-data Jacobian)            */
    double gemm_flops;           /* the useful flops of those calls (part of contract_flops)   */
} dot_stats;

const char* dot_version(void);
/* Text of the last error on this problem (or of the last failed dot_create if P is NULL). */
const char* dot_last_error(const dot_problem* P);

/* Create a problem on the current CUDA device.  No device memory is allocated
 * until dot_bind_workspace.  Errors: DOT_ERR_ARG (sizes, node indices out of
 * range, duplicate nodes on one side). */
int dot_create(const dot_config* cfg, dot_problem** out);
int dot_destroy(dot_problem* P);

/* All work of P is enqueued on `cuda_stream` (a cudaStream_t; NULL = legacy default). */
int dot_set_stream(dot_problem* P, void* cuda_stream);

/* Device bytes for the persistent state plus `max_rhs` simultaneously iterated
 * right-hand sides.  Larger requests are processed in
 * chunks of what fits. */
size_t dot_workspace_bytes(const dot_problem* P, int32_t max_rhs);
/* Bind caller-owned device memory (>= dot_workspace_bytes(P, 1)).  Rebinding
 * invalidates parameters, data and cached fields. */
int dot_bind_workspace(dot_problem* P, void* dev_ptr, size_t bytes);
/* Enable CUDA-event timing of the CG pass and contraction kernels (dot_stats). */
int dot_enable_timing(dot_problem* P, int on);
int dot_get_stats(const dot_problem* P, dot_stats* out);
int dot_reset_stats(dot_problem* P);

/* Measured data D_f (Eq. (3.1)): [n_freq][n_det][n_src] complex. */
int dot_set_data(dot_problem* P, const double* data, int where);

/* ---- paper-level calls (BASELINE north_star: set_params, misfit, jacobian, optimize_directions) */

/* set_params(p): p = [n_p] = per basis (alpha, beta, chi_x, chi_y, chi_z)
 * (Eq. (2.3)).  Evaluates mu(x, p) (Eq. (2.4)), the support S of
 * dA/dp and G = theta dmu/dp on S (L972), and invalidates cached fields. */
int dot_set_params(dot_problem* P, const double* p, int where);

/* misfit(W, V): solves A(omega_f) z_i = B w_i for the ls simultaneous sources
 * of every frequency (PAPER.md Eq. (EsTResidual)) -- unless cached --
 * and returns
 *   misfit_out (host) = sum_f || V^T (C^T Z_f - D_f W) ||_F^2      (Eq. (3.12)),
 *   resid_out  [n_freq][ld][ls] complex = V^T R_f W   (may be NULL).
 * W: [n_src][ls] row-major real, or NULL for W = I (ls must be n_src).
 * V: [n_det][ld] row-major real, or NULL for V = I (ld must be n_det).
 * The forward fields are kept (sampled on P = S u detectors u sources) for dot_jacobian.
 * Errors: DOT_ERR_STATE (no params / no data), DOT_ERR_NOCONV, DOT_ERR_BREAKDOWN. */
int dot_misfit(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld,
               int where, double* misfit_out, double* resid_out);

/* jacobian(W, V): J_out [n_freq][ld][ls][n_p] complex,
 *   J[f][j][i][k] = - y_j^T diag(G_k) z_i,  z_i = A_f^-1 B w_i,  y_j = A_f^-T C v_j
 * (Eqs. (2.8), (3.12), (Jacobian kth column) L966-972).  Forward fields
 * come from the cache of a preceding dot_misfit/dot_jacobian with the same W (or
 * by linear combination of cached full-data fields), else are solved; the ld
 * adjoint solves likewise.  The contraction is block-sparse by basis (L972: only the
 * points where dA/dp_k != 0 enter): panels of ld >= 32 rows and ls >= 8 columns run as a
 * 3-multiply complex GEMM per (frequency, basis) on FP64 tensor cores (DMMA); small sketched
 * panels (ld * ls <= 256) as FP64 FMA partial sums over k-tiles with a fixed-order reduction.
 * Scratch (operand tiles, partials) comes from the bound workspace: DOT_ERR_WORKSPACE if
 * it cannot hold one frequency's operand tiles for one column tile. */
int dot_jacobian(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld,
                 int where, double* J_out);

/* optimize_directions(k): replace k simultaneous random sources and k detectors
 * by simultaneous optimized ones (Sec. 3.2-3.3.2, Theorems 3.4-3.7):
 * phase one alternately removes one source then one detector, phase two
 * alternately adds one source then one detector.  Needs the full-data fields
 * (n_src + n_det solves per frequency, cached).  W_out [n_src][ls],
 * V_out [n_det][ld]; the first ls-k (ld-k) columns span a subspace of the input
 * columns, the last k are the optimized directions scaled to length sqrt(n).
 * objective_out (host, may be NULL): ||(W_out^T (x) V_out^T) J||_F^2. */
int dot_optimize_directions(dot_problem* P, int32_t k, const double* W, int32_t ls,
                            const double* V, int32_t ld, int where,
                            double* W_out, double* V_out, double* objective_out);

/* optimize_directions by subspace iteration (reading R16; BASELINE.json
 * configs[3] "optimized ... found by 5 subspace iterations maximizing ||V^T J W||_F"):
 * same two-phase replacement as dot_optimize_directions, but the add steps
 * (Theorems 3.7, 3.6) find the new direction by `iters` steps of
 * subspace iteration with a `block`-vector block on P Xr Xr^T P, applied matrix-free
 * (2 n_freq solves per block vector per step) -- no full-data solves.  The remove
 * steps (Theorems 3.5, 3.4) use the sketched Jacobian of the current W, V
 * (ls + ld solves per frequency, combined without new solves afterwards).
 * X0_src [n_src][k*block], X0_det [n_det][k*block]: starting blocks (the caller's
 * random draws); add step t starts from columns t*block .. (t+1)*block - 1.  New columns: unit direction with
 * its largest-magnitude entry positive, scaled to length sqrt(n).  Errors as
 * dot_optimize_directions; DOT_ERR_ARG if block exceeds the complement dimension. */
int dot_optimize_directions_subspace(dot_problem* P, int32_t k, int32_t iters, int32_t block, const double* W,
                                     int32_t ls, const double* V, int32_t ld, const double* X0_src,
                                     const double* X0_det, int where, double* W_out, double* V_out,
                                     double* objective_out);

/* ---- z-slab domain decomposition (BASELINE north_star: "by z-slab domain decomposition
 * with NCCL halo exchange and an allreduce of Krylov inner products in the few-
 * simultaneous-source regime").  Rank r of `world`
 * owns a contiguous range of z chunks and iterates only those planes (plus the halo
 * planes it recomputes); after every CG pass the two boundary planes of r_{k+1} and
 * p_k of every seed pair are packed into ONE buffer per neighbour, exchanged, and the
 * per-chunk partial sums of the Krylov inner products are summed over the ranks, so
 * all ranks take identical steps.  Each rank folds the shifted solutions on its own
 * samples; they are summed over the ranks at the end and land in each rank's field
 * caches, after which dot_misfit / dot_jacobian / dot_solve_sampled on any rank use
 * them without solves.
 *
 * Three transports, one code path:
 *  - all ranks in this process (nlocal == world): device copies (single-GPU emulation);
 *  - one rank per process with NCCL (nlocal == 1, nccl_id): ncclSend/ncclRecv of the
 *    packed halo buffers, ncclAllReduce of the partials;
 *  - one rank per process with a caller transport (dot_dd_create_transport): the packed
 *    buffers are staged through host memory and handed to the caller's callbacks, e.g.
 *    torch.distributed point-to-point and all_reduce over a gloo group.
 *
 * dot_nccl_unique_id: 128-byte NCCL id (host); rank 0 creates it, the caller
 *   broadcasts it (e.g. torch.distributed).  NCCL is loaded at run time.
 * dot_dd_create: `local` [nlocal] problems of ranks rank0 .. rank0+nlocal-1.  Either
 *   nlocal == world (in-process) or nlocal == 1 with nccl_id (one rank per process; world 1
 *   with an id runs the NCCL path on one GPU: all-reduces, no neighbours).  All ranks hold
 *   the same problem and parameters (dot_set_params on each).
 * dot_transport: sendrecv(ctx, peer, send, send_bytes, recv, recv_bytes) exchanges host
 *   buffers with rank `peer` (the peer calls it with the mirrored sizes; either size may be
 *   0); allreduce_sum(ctx, buf, n) sums n doubles in place over all ranks.  Both return 0
 *   on success.  Called on the thread that called dot_dd_fields, buffers owned by the
 *   library and valid for the duration of the call.
 * dot_dd_fields: solve the forward fields of B W (ls columns; W NULL = identity;
 *   ls = 0: none) and the adjoint fields of C V (ld; likewise) for every frequency
 *   in one decomposed batch and cache them on every local rank.  Errors as
 *   dot_misfit; DOT_ERR_ARG if nz < 2 * world; DOT_ERR_CUDA if a transport call fails. */
typedef struct dot_transport {
    void* ctx;
    int (*sendrecv)(void* ctx, int32_t peer, const void* send, size_t send_bytes, void* recv, size_t recv_bytes);
    int (*allreduce_sum)(void* ctx, double* buf, size_t n);
} dot_transport;
int dot_nccl_unique_id(unsigned char* id_out);
int dot_dd_create(dot_problem* const* local, int32_t nlocal, int32_t rank0, int32_t world,
                  const unsigned char* nccl_id, dot_dd** out);
int dot_dd_create_transport(dot_problem* local, int32_t rank, int32_t world, const dot_transport* t, dot_dd** out);
int dot_dd_fields(dot_dd* G, const double* W, int32_t ls, const double* V, int32_t ld, int where);
const char* dot_dd_last_error(const dot_dd* G);
int dot_dd_destroy(dot_dd* G);

/* prefetch_fields(W, V): solve the forward fields of B W (ls columns; W NULL =
 * identity; ls = 0: none) and the adjoint fields of C V (ld; likewise) that are not
 * already cached, all frequencies, in ONE batch (L966: "we solve A(p) z_i = B w_i ...
 * A^T(p) y_j = C v_j"), so that a following dot_misfit / dot_jacobian /
 * dot_fields_on_support with these W, V runs without solves. */
int dot_prefetch_fields(dot_problem* P, const double* W, int32_t ls, const double* V, int32_t ld, int where);

/* ---- component calls (same kernels; used by the parity tests) ---- */

/* mu(x, p) of the last set_params: mu_out [N] real. */
int dot_absorption(dot_problem* P, double* mu_out, int where);
/* Support of dA/dp: K_out (host) = |S|; if nodes_out/G_out are non-NULL they
 * receive S (ascending node indices, [K] int64) and G = theta dmu/dp on S
 * ([K][n_p] row-major). */
int dot_support(dot_problem* P, int32_t* K_out, int64_t* nodes_out, double* G_out, int where);
/* Au = A(omega_f, p) u for nrhs fields: u, Au [nrhs][N] complex. */
int dot_apply(dot_problem* P, int32_t freq, int32_t nrhs, const double* u, double* Au, int where);
/* Solve A(omega_{freq[r]}, p) x_r = b_r (Eq. (2.1)) with the multi-shift CG kernels
 * (Re b_r and Im b_r are two real seeds at shift omega_{freq[r]}/nu, every node sampled):
 * b, x [nrhs][N] complex; freq [nrhs] int32 (same `where`).  iters_out (host, may be NULL)
 * [nrhs]: iterations of the slower seed.  Dense-output test/diagnostic call: the workspace
 * of dot_workspace_bytes covers up to 3 right-hand sides per call. */
int dot_solve(dot_problem* P, int32_t nrhs, const int32_t* freq, const double* b, double* x,
              int where, int32_t* iters_out);
/* Sampled solve of point-source / point-detector combinations: side 0 = sources
 * (rhs = B w), 1 = detectors (rhs = C v); coeff [n_side][ncols] real (NULL = I);
 * for every frequency.  X_out [n_freq][ncols][n_samples] complex holds the
 * solution on the sample nodes P (dot_samples), solved fields are cached. */
int dot_solve_sampled(dot_problem* P, int32_t side, const double* coeff, int32_t ncols,
                      int where, double* X_out);
/* Same fields restricted to the support S of dA/dp (the Jacobian's only
 * consumers, L972): out [n_freq][ncols][K] complex, K = |S| in dot_support
 * order.  Fields of combinations of already-solved point sources (identity or
 * selection caches) are formed by linear combination without new solves;
 * multi-GPU callers all-reduce these partial combinations. */
int dot_fields_on_support(dot_problem* P, int32_t side, const double* coeff, int32_t ncols, int where,
                          double* out);
/* Sample nodes P = S u detectors u sources (ascending, [n_samples] int64). */
int dot_samples(dot_problem* P, int32_t* n_out, int64_t* nodes_out, int where);

/* Jacobian contraction of explicit field panels on P's support S with P's weights
 * (block-sparse by basis when available, as dot_jacobian):
 *   J[f][j][i][k] = - sum_s Lam[f][j][s] U[f][i][s] G[s][k]
 * Lam [n_freq][ld][K], U [n_freq][ls][K], J [n_freq][ld][ls][n_p] complex, DEVICE
 * pointers (K = |S| of the last set_params).  Used by the multi-GPU step on
 * all-reduced / all-gathered fields.  Counts in dot_stats like dot_jacobian. */
int dot_contract_fields(dot_problem* P, int32_t ld, int32_t ls, const double* Lam, const double* U, double* J);

/* Stateless Jacobian contraction on explicit panels (no problem needed):
 *   J[b][j][i][k] = - sum_s Lam[b][j][s] U[b][i][s] G[s][k]
 * Lam [nb][ld][K], U [nb][ls][K] complex, G [K][n_p] real, J [nb][ld][ls][n_p]
 * complex.  Runs the DMMA kernel on `cuda_stream`; all arrays DEVICE pointers,
 * 16-byte aligned; n_p <= 256.  Algorithmic flops: 4 nb ld ls K n_p. */
int dot_contract(void* cuda_stream, int32_t nb, int32_t K, int32_t ld, int32_t ls, int32_t n_p,
                 const double* Lam, const double* U, const double* G, double* J);

/* Host utility (no GPU): eigen-decomposition of a dense symmetric n x n matrix
 * A (row-major), used for the small SVD problems of PAPER.md Table 1 via
 * Lemma 3.2 (left singular vectors of M are the eigenvectors of M M^T).
 * w [n] eigenvalues in descending order, Z [n][n] row-major with the
 * eigenvectors as columns.  Returns 0, or 1 if the QL iteration failed. */
int dot_sym_eig(int n, const double* A, double* w, double* Z);

#ifdef __cplusplus
}
#endif
#endif /* DOT_B200_H */
