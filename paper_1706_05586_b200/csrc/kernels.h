// Kernel launchers of the B200 DOT library (internal interface between the
// C-ABI layer abi.cu and the kernel translation units).
#pragma once
#include "dot_common.cuh"

namespace dot {

// ------------------------------------------------------------------ cocg.cu
// Tiling of the fused COCG pass: a CTA owns TY full x-rows of one RHS and
// marches all nz planes; planes (with a 2-row y halo) are staged by TMA bulk
// copies into a ring of `nslots` shared-memory slots.
struct CocgTiling {
    int kind = 1;         // 1: z-register pass (cocg_z.cu), 0: padded-ring pass (cocg.cu)
    int cluster = 1;      // thread-block cluster size along the tiles of one RHS (divides ntiles)
    int minb = 1;         // CTAs per SM the z pass is compiled for
    int zrows = 1;        // z pass: slot rows per thread (1 or 2)
    int TY = 0, ntiles = 0, nslots = 0, threads = 512;
    int rpt = 0;          // x-rows covered by one sweep of the block (threads = roundup32(nx * rpt))
    size_t smem = 0;
};
// prefetch: planes loaded ahead (slots = prefetch + 3); max_smem: per-CTA budget (bytes)
// kind: 1 = z-register pass if a tiling fits (else the ring pass), 0 = ring pass;
// want_ty > 0 forces the z-pass tile height.
CocgTiling cocg_tiling(int nx, int ny, int nz, int prefetch = 1, size_t max_smem = 0, int max_threads = 0,
                       int kind = 1, int want_ty = 0);

struct PassArgs {
    OpConst op;
    CocgTiling tl;
    int k = 0;                    // pass index
    int nzch = 1;                 // z chunks launched per (tile, RHS) (z pass only)
    int zlen = 0;                 // planes per z chunk
    int zc0 = 0;                  // first (global) z chunk of this launch (z-slab domain decomposition)
    int nzch_tot = 1;             // global z chunks: partial slots per RHS = ntiles * nzch_tot
    const int32_t* act = nullptr; // z pass: grid row y iterates RHS act[y] (active list), null = identity
    int max_iter = 0;
    double tol2 = 0;              // tol^2
    const double* mu = nullptr;   // [N] absorption
    const double* shift = nullptr;// [nb] omega/nu of each RHS
    double2* R[2] = {nullptr, nullptr};   // [nb][N] residual r (ping-pong)
    double2* Pv[2] = {nullptr, nullptr};  // [nb][N] direction p (ping-pong)
    double* part[2] = {nullptr, nullptr}; // [nb][ntiles][kNumPartials]
    RhsState* st[2] = {nullptr, nullptr}; // [nb]
    const int32_t* samp_nodes = nullptr;  // [nP] ascending node ids
    const int32_t* samp_off = nullptr;    // [nz*ntiles+1] ranges of samples per (plane, tile)
    double2* XP = nullptr;                // [nb][nP] sampled solution
    int nP = 0;
    double2* X = nullptr;                 // [nb][N] full solution (test mode) or null
};

// Launch a pass kernel, as a thread-block cluster of `cs` consecutive tiles of one
// RHS when cs > 1 (co-scheduled, so y-halo rows read by neighbours hit in L2).
template <class K>
void launch_clustered(K kernel, dim3 grid, int threads, size_t smem, cudaStream_t s, int cs, const PassArgs& a) {
    if (cs <= 1) {
        kernel<<<grid, threads, smem, s>>>(a);
    } else {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = grid;
        cfg.blockDim = dim3(threads);
        cfg.dynamicSmemBytes = smem;
        cfg.stream = s;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        DOT_CUDA_TRY(cudaLaunchKernelEx(&cfg, kernel, a));
    }
    DOT_CUDA_TRY(cudaGetLastError());
}

// z-register pass (cocg_z.cu)
size_t zpass_smem(int nx, int TY, int NS, int nz);
void launch_cocg_zpass(const PassArgs& a, int nb, cudaStream_t s);
void launch_cocg_init(const PassArgs& a, int nb, cudaStream_t s);
void launch_cocg_pass(const PassArgs& a, int nb, cudaStream_t s);
// *d_count = number of RHS not done; act (optional, [nb]) receives their indices in order
void launch_count_active(const RhsState* st, int nb, int* d_count, cudaStream_t s, int32_t* act = nullptr);
void launch_apply(const OpConst& op, const double* mu, const double* shift, const double2* u,
                  double2* Au, int nb, cudaStream_t s);
// Chunk of the global RHS list r = f*ncols + c (r = rg0 .. rg0+nb-1):
// R0[r][node[a]] = coeff[a*ncols + c] * scale[a]  (coeff == null: identity)
void launch_scatter_rhs(double2* R0, size_t N, int nb, long long rg0, int ncols, const int32_t* nodes,
                        int nnodes, const double* coeff, const double* scale, cudaStream_t s);
// shift[r] = omega_over_nu[(rg0 + r) / ncols]
void launch_fill_shift(double* shift, int nb, long long rg0, int ncols, const double* omega_over_nu,
                       cudaStream_t s);

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
};
// sp == null (or no segments): dense DMMA contraction over all K points; else the
// block-sparse one (per basis j, its support points only).
void launch_contract(int nb, int K, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                     const double2* U, size_t u_bstride, const double* G, double2* J,
                     cudaStream_t s, const GSparse* sp = nullptr);
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
