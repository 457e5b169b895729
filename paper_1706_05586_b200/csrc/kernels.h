// Kernel launchers of the B200 DOT library (internal interface between the
// C-ABI layer abi.cu and the kernel translation units).
#pragma once
#include <cuda.h>

#include "dot_common.cuh"

namespace dot {

class Arena;

// ------------------------------------------------------------------ cg_shift.cu
// Tiling of the fused multi-shift CG pass: a CTA owns TY full x-rows of one pair of real
// seeds and marches the nz planes; planes (with a 2-row y halo) are staged by TMA bulk
// copies into a ring of `nslots` shared-memory slots.
struct CgTiling {
    int rows = 2;         // slot rows per thread (1 or 2)
    bool mut = true;      // mu rides in the ring slots (TMA); else per-thread loads from L2
    int TY = 0, ntiles = 0, nslots = 0, threads = 512;
    int xs = 1;           // x parts per row tile (wide rows); ntiles = nty * xs CTA tiles
    int nxl = 0;          // slot row width: nx (xs = 1) or ceil(nx / xs) + 4 (2 halo columns per side)
    int nty = 0;          // row tiles (sample offsets are per (plane, row tile))
    size_t smem = 0;
    bool pdl = true;      // passes launched with programmatic stream serialization (DOT_CG_PDL=0: plain)
};
// prefetch: planes loaded ahead (1..3; slots = prefetch + 2); want_ty > 0 forces the tile height,
// want_rows > 0 the rows per thread
// want_xs > 0 forces the x parts (1 or 2).
CgTiling cg_tiling(int nx, int ny, int nz, int prefetch = 2, int want_ty = 0, int want_rows = 0, bool no_mu = false,
                   int want_xs = 0);
size_t pass_smem(int nx, int TY, int NS, int nz, bool mut);

struct PassArgs {
    OpConst op;
    CgTiling tl;
    int k = 0;                    // pass index
    int nzch = 1;                 // z chunks launched per (tile, pair)
    int zlen = 0;                 // planes per z chunk
    int zc0 = 0;                  // first (global) z chunk of this launch (z-slab domain decomposition)
    int nzch_tot = 1;             // global z chunks: partial slots per pair = ntiles * nzch_tot
    const int32_t* act = nullptr; // grid row y iterates pair act[pair0 + y] (active list), null = identity
    int pair0 = 0;                // first grid row of this launch (a batch split over two streams)
    int max_iter = 0;
    double tol2 = 0;              // tol^2
    int nshift = 0;               // frequencies (shifts i omega_f / nu of the scaled system)
    double sigma[kMaxShift] = {}; // omega_f / nu
    double ec[4][3] = {};         // K~ coefficients (diagonal, down, up) of planes 0, 1, nz-2, nz-1
    const double* mu = nullptr;   // [N] absorption
    double2* R[2] = {nullptr, nullptr};   // [npairs][N] residual r~ of two real seeds (ping-pong)
    double2* Pv[2] = {nullptr, nullptr};  // [npairs][N] direction p~ (ping-pong)
    double* part[2] = {nullptr, nullptr}; // [npairs][nzch_tot][ntiles][kNumPartials]
    SeedState* st[2] = {nullptr, nullptr};// [2 npairs]
    ShiftState* sh[2] = {nullptr, nullptr};// [2 npairs][kMaxShift]
    const uint32_t* mask = nullptr;       // [2 npairs] shifts each seed must deliver
    ShiftCoef* coef = nullptr;            // [hist][2 npairs][kMaxShift]
    int hist = kHist;                     // depth of the coef / H rings (passes between folds)
    int npairs = 0;                       // pairs of the batch (strides of coef / H)
    const int32_t* samp_nodes = nullptr;  // [nP] ascending node ids
    const int32_t* samp_off = nullptr;    // [nz*ntiles+1] ranges of samples per (plane, tile)
    int nP = 0;
    double2* H = nullptr;                 // [hist][npairs][nP] seed residual r_k at the samples
    // x split (tl.xs > 1): the slot tiles arrive as one tensor copy per vector (rows and columns
    // outside the domain zero-filled by the copy).  R[i] / Pv[i] as [pair][z][y][2 nx] doubles,
    // mu as [z][y][nx]; boxes of (TY + 4) rows x nxl columns.  Filled by set_pass_tmaps.
    CUtensorMap tmR[2], tmP[2], tmMu;
};
// encodes PassArgs::tmR / tmP / tmMu from R, Pv, mu, op, tl, npairs (no-op when tl.xs == 1)
void set_pass_tmaps(PassArgs& a);

struct FoldArgs {
    int k0 = 0, k1 = 0;                   // passes to fold
    int s0 = 0, s1 = 0;                   // sample range
    int npairs = 0, nshift = 0, nP = 0;
    int hist = kHist;                     // ring depth
    int nsl = 0;                          // shift slots per seed (needed shifts in ascending order)
    const uint32_t* mask = nullptr;
    const ShiftCoef* coef = nullptr;
    const double2* H = nullptr;
    double2* Ps = nullptr;                // [2 npairs][nsl][nP] shifted directions on the samples
    double2* Xs = nullptr;                // [2 npairs][nsl][nP] shifted solutions (scaled variables)
};

// fills PassArgs::ec from PassArgs::op (call after setting op)
void set_edge_coefs(PassArgs& a);
void launch_cg_pass(const PassArgs& a, int nb, cudaStream_t s);
// zc_own: the z-chunk slot that carries the initial sums (0)
void launch_cg_init(const PassArgs& a, int nb, cudaStream_t s, int zc_own = 0);
void launch_cg_fold(const FoldArgs& f, cudaStream_t s);
// omap[3 seed] = (output base, output stride per shift, 1 if the seed is the imaginary part)
void launch_cg_finalize(const FoldArgs& f, const OpConst& op, double2* XP, int nP_out, const int32_t* omap,
                        const int32_t* samp_nodes, cudaStream_t s);
// *d_count = number of pairs with a seed not done; act (optional, [npairs]) receives them in order
void launch_count_active(const SeedState* st, int npairs, int* d_count, cudaStream_t s, int32_t* act = nullptr);
// A(omega, p) u in the original variables (dot_apply)
void launch_apply(const OpConst& op, const double* mu, const double* shift, const double2* u,
                  double2* Au, int nb, cudaStream_t s);
// chunk-local seeds seed0 .. seed0+nseeds-1 (pair = seed / 2, component = seed % 2) are the
// columns col0 .. of one segment: R0[pair][node[a]] = coeff[a*ncols + col] * scale[a] * theta^-1/2
// (coeff null: identity)
void launch_scatter_seeds(double2* R0, size_t N, const int32_t* nodes, int nnodes, const double* coeff, int ncols,
                          const double* scale, int col0, int seed0, int nseeds, const OpConst& op, cudaStream_t s);
// z-slab halo planes z0 .. z0+n-1 of r and p of every pair <-> buf [2][npairs][n][PS]
void launch_pack_planes(const double2* R, const double2* Pv, int npairs, size_t N, int PS, int z0, int n,
                        double2* buf, cudaStream_t s);
void launch_unpack_planes(double2* R, double2* Pv, int npairs, size_t N, int PS, int z0, int n, const double2* buf,
                          cudaStream_t s);
// dense complex RHS r -> pair r = (Re, Im) * theta^-1/2
void launch_split_dense(double2* R0, const double2* b, size_t N, int nr, const OpConst& op, cudaStream_t s);

// ------------------------------------------------------------------ pals.cu
struct PalsConst {
    int nx, ny, nz, n_rbf;
    double hx, hy, hz, gamma, eps, cutoff, mua_in, mua_out;
};
// mu[N], flagS[N] (1 where dH/dphi != 0), flagP[N] = flagS | detector
void launch_pals_eval(const PalsConst& c, const double* params, double* mu, int32_t* flagS,
                      int32_t* flagP, cudaStream_t s);
void launch_mark_nodes(int32_t* flag, const int32_t* nodes, int n, cudaStream_t s);
// exclusive scan of int32 flags -> pos (int32), total -> *d_total
size_t scan_temp_bytes(size_t n);
void launch_exclusive_scan(const int32_t* in, int32_t* out, size_t n, int32_t* d_total, void* temp,
                           cudaStream_t s);
void launch_compact(const int32_t* flag, const int32_t* pos, size_t n, int32_t* out_nodes,
                    cudaStream_t s);
void launch_gather_rank(const int32_t* pos, const int32_t* nodes, int n, int32_t* out, cudaStream_t s);
// G[s][k] = theta dmu/dp_k at S[s]
void launch_pals_grad(const PalsConst& c, const double* params, const int32_t* S, int K, double* G,
                      cudaStream_t s);
void launch_sample_offsets(const int32_t* P, int nP, int nx, int ny, int nz, int TY, int ntiles,
                           int32_t* off, cudaStream_t s);

// ------------------------------------------------------------------ contract.cu
// Block sparsity of G by RBF ("we first find the few nonzero components
// of dA/dp_k"): seg[segoff[j] .. segoff[j+1]) lists the support points (indices into S,
// ascending) where the 5 parameters of basis j have nonzero weights.
struct GSparse {
    const int32_t* seg = nullptr;
    const int32_t* segoff = nullptr;   // [n_rbf + 1]
    int n_rbf = 0;
    long long total = 0;               // segoff[n_rbf]
    // k-tiles of 16 basis-ordered points that never straddle two bases (contract_seg_tma,
    // contract_small): ktile[g] = (first point, end of its basis's points, basis j, 0),
    // kto[j] = first k-tile of basis j
    const int4* ktile = nullptr;
    const int32_t* kto = nullptr;      // [n_rbf + 1]
    int ktiles = 0;                    // kto[n_rbf]
    const int32_t* jorder = nullptr;   // [n_rbf] bases by decreasing k-tile count (work order)
    int maxkt = 0;                     // largest k-tile count of one basis
};
// sp == null (or no segments): dense DMMA contraction over all K points; else the
// block-sparse one (per basis j, its support points only).
// With `arena` and small panels (ld * ls <= 256: the sketched / optimized-direction shapes) the
// block-sparse form runs split over the k-tiles (contract_small_kernel) with a fixed-order
// reduction; launches are added to *launches when given.
void launch_contract(int nb, int K, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                     const double2* U, size_t u_bstride, const double* G, double2* J,
                     cudaStream_t s, const GSparse* sp = nullptr, Arena* arena = nullptr,
                     int64_t* launches = nullptr);
// Block-sparse GEMM on basis-ordered panels (the default for large panels): Lam [nb][ld][T],
// U [nb][ls][T] with column t the support point seg[t] of basis j (segoff[j] <= t < segoff[j+1]),
// Gs [T][5] the basis's weights there.  contract_seg_applies: the panel shape takes this path.
bool contract_seg_applies(int ld, int ls, const GSparse* sp, int n_p);
// The GEMM runs through pre-formed operand tiles: per frequency, a prescale pass
// writes the 3-multiply operands (A = Lam, B = Gs U as (re, im) + (re + im) planes) as
// 64-row x 16-point blocks in the exact shared-memory image the GEMM consumes; the GEMM
// streams them with one cp.async.bulk per block into a 4-stage mbarrier ring and runs LDS +
// DMMA only.  Operand tiles come from `arena` (chunked over column tiles when it is short);
// launches are added to *launches.
void contract_seg_tma(int nb, int T, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                      const double2* U, size_t u_bstride, const double* Gs, const GSparse& sp, double2* J,
                      Arena& arena, cudaStream_t s, int64_t* launches, double* dmma_flops = nullptr);
// bytes of one frequency's operand tiles (the workspace estimate)
size_t contract_seg_tma_bytes(int ld, int ls, long long total, int n_rbf);
// Gs[t][q] = G[seg[t]][5 j + q]
void launch_seg_weights(const double* G, int n_p, const GSparse& sp, double* Gs, cudaStream_t s);
// idx[t] = slot[seg[t]]
void launch_compose_index(const int32_t* seg, int T, const int32_t* slot, int32_t* idx, cudaStream_t s);
// flags F[j][s] = any(G[s][5j .. 5j+4] != 0), j < n_rbf
void launch_rbf_flags(const double* G, int K, int n_rbf, int32_t* F, cudaStream_t s);
// out[pos[i]] = i % K for flagged i (segment lists), off[j] = pos[j*K], off[n_rbf] = *total
void launch_rbf_segments(const int32_t* F, const int32_t* pos, int K, int n_rbf, const int32_t* total,
                         int32_t* seg, int32_t* off, cudaStream_t s);

// ------------------------------------------------------------------ smallops.cu
// out[b][m][n] = sum_k Rm[k*ldr + m] * Cx[b*sb + k*sk + n*sn]   (real^T x complex)
void launch_rc_gemm(int nb, int M, int N, int K, const double* Rm, int ldr, const double2* Cx,
                    size_t sb, size_t sk, size_t sn, double2* out, size_t ob, size_t om, size_t on,
                    cudaStream_t s);
// out[b][i][j] = X[b][i][idx[j]] (gather columns)
void launch_gather_cols(int nb, int rows, int ncols, const double2* X, size_t xb, size_t xr,
                        const int32_t* idx, double2* out, size_t ob, size_t orow, cudaStream_t s);
// X[r][c] *= scale[c] (complex X [rows][ncols], real scale)
void launch_scale_cols(double2* X, size_t rows, int ncols, const double* scale, cudaStream_t s);
// a[i] -= b[i] (complex)
void launch_csub_inplace(double2* a, const double2* b, size_t n, cudaStream_t s);
// a[i] += b[i] (complex)
void launch_cadd_inplace(double2* a, const double2* b, size_t n, cudaStream_t s);
// *out = sum |a[i]|^2 (deterministic, single launch)
void launch_sumsq(const double2* a, size_t n, double* out, cudaStream_t s);
// Dt[f][s][d] = D[f][d][s]
void launch_transpose_data(const double2* D, int nf, int nd, int ns, double2* Dt, cudaStream_t s);

// R[r][S[x]] = w[r][x], r < nr (dense right-hand sides supported on S)
void launch_scatter_support(double2* R, size_t N, int nr, const int32_t* S, int K, const double2* w, cudaStream_t s);
// w[f][q][x] = sum_i Z[f][i][x] sum_k C[f][q][i][k] G[x][k]   (C [nf][nq][ncol][n_p], Z [nf][ncol][K])
void launch_form_support_rhs(int nf, int nq, int K, int ncol, int n_p, const double2* C, const double2* Z,
                             const double* G, double2* w, cudaStream_t s);

}  // namespace dot
