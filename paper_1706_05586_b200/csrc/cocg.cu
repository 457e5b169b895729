// Batched multi-RHS COCG for the complex-symmetric DOT operator A(omega, p)
// (Eq. (2.1), Eq. (2.5); solves of Sec. 3.3.1 "we solve
// A(p) z_i = B w_i ... A^T(p) y_j = C v_j").
//
// Single-pass COCG: the state carried between passes is
// (r_k, p_{k-1}) plus per-RHS scalars.  Pass k forms p_k = r_k + beta_k p_{k-1},
// q_k = A p_k, r_{k+1} = r_k - alpha_k q_k and, in the same sweep, the reductions
// rho_{k+1} = r^T r, mu_{k+1} = r^T A r, nu_{k+1} = r^T q_k and the direct
// sigma_k = p_k^T q_k.  The next pass takes beta_{k+1} = rho_{k+1}/rho_k,
// sigma_{k+1} = mu_{k+1} + 2 beta nu_{k+1} + beta^2 sigma_k, alpha = rho/sigma.
// HBM traffic per point and iteration: read r, p; write r, p = 64 B.
#include <cstdlib>
#include <vector>

#include "kernels.h"

namespace dot {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block reduction of kNumPartials doubles; result valid in thread 0.
__device__ void block_reduce_partials(double (&acc)[kNumPartials], double* scratch) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) acc[i] = warp_sum(acc[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < kNumPartials; ++i) scratch[warp * kNumPartials + i] = acc[i];
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kNumPartials; ++i) {
            double s = 0;
            for (int w = 0; w < nw; ++w) s += scratch[w * kNumPartials + i];   // fixed order
            acc[i] = s;
        }
    }
}

struct Scalars {
    double2 alpha, beta;
    int active;   // 0: exit
};

// Scalar recurrences at the start of pass k (identical in every CTA of one RHS).
__device__ Scalars pass_scalars(const PassArgs& a, int rhs, int tile) {
    const int ntiles = a.tl.ntiles;
    const RhsState prev = a.st[(a.k + 1) & 1][rhs];
    RhsState cur = prev;
    Scalars sc;
    sc.alpha = cmk(0, 0);
    sc.beta = cmk(0, 0);
    sc.active = 0;
    if (!prev.done) {
        const double* pp = a.part[a.k & 1] + (size_t)rhs * ntiles * kNumPartials;
        double s[kNumPartials];
        for (int i = 0; i < kNumPartials; ++i) s[i] = 0;
        for (int t = 0; t < ntiles; ++t)
            for (int i = 0; i < kNumPartials; ++i) s[i] += pp[t * kNumPartials + i];
        const double2 rho = cmk(s[0], s[1]), mu = cmk(s[2], s[3]), nu = cmk(s[4], s[5]);
        const double2 sigd = cmk(s[6], s[7]);
        const double nrm2 = s[8];
        if (a.k == 0) cur.bnorm2 = nrm2;
        double2 beta = cmk(0, 0), sigma = mu;
        if (a.k > 0) {
            beta = cdiv(rho, cmk(prev.rho_re, prev.rho_im));
            sigma = cadd(cadd(mu, cscale(cmul(beta, nu), 2.0)), cmul(cmul(beta, beta), sigd));
        }
        const double2 alpha = cdiv(rho, sigma);
        if (!(nrm2 > a.tol2 * cur.bnorm2)) {           // converged (also b = 0)
            cur.done = 1;
            cur.iters = a.k;
        } else if (a.k >= a.max_iter) {
            cur.done = 1;
            cur.iters = a.k;
            cur.flag = DOT_ERR_NOCONV;
        } else if (!isfinite(alpha.x) || !isfinite(alpha.y) || !isfinite(beta.x) ||
                   !isfinite(beta.y)) {
            cur.done = 1;
            cur.iters = a.k;
            cur.flag = DOT_ERR_BREAKDOWN;
        } else {
            sc.active = 1;
            sc.alpha = alpha;
            sc.beta = beta;
            cur.rho_re = rho.x;
            cur.rho_im = rho.y;
            cur.alpha_re = alpha.x;
            cur.alpha_im = alpha.y;
        }
    }
    if (tile == 0) a.st[a.k & 1][rhs] = cur;
    return sc;
}

// One fused COCG pass.  grid = (ntiles, nb), block = tl.threads.
// Shared memory: NS plane slots for r_k and p_{k-1} -> p_k ([TY+4 rows][nx+2] with zero
// guard columns = Dirichlet x-faces, zero rows outside the y-range), and a ring of 3
// r_{k+1} planes ([TY+2][nx+2]).  Step f of the z-march:
//   A  bulk copies of plane f+PD into smem (warp 0); L2 prefetch of plane f+LPD (warp 1)
//   B  p_k(f) = r_k(f) + beta p_{k-1}(f); write p_k(f) rows    (phase 1)
//      A r_{k+1} at plane f-3, reductions, write r_{k+1}(f-3)  (phase 3)
//   -- barrier --
//   C  q = A p_k at plane f-1, r_{k+1}(f-1) = r_k - alpha q, reductions, samples
//   -- barrier --
// Template parameters fix the geometry at compile time (0 = read at run time).
template <bool FULLX, int NX_, int TY_, int NS_, int RPT_>
__global__ void __launch_bounds__(512, 1) cocg_pass_kernel(const PassArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int MAXR = 4;                       // rows per thread per phase (tiling guarantees)
    constexpr int LPD = 4;                        // L2 prefetch distance (planes)
    const int tile = blockIdx.x, rhs = blockIdx.y;
    const int nx = NX_ ? NX_ : a.op.nx;
    const int ny = a.op.ny, nz = a.op.nz;
    const int TY = TY_ ? TY_ : a.tl.TY;
    const int NS = NS_ ? NS_ : a.tl.nslots;
    const int RPT = RPT_ ? RPT_ : a.tl.rpt;
    const int ntiles = a.tl.ntiles;
    const int W = nx + 2;                          // padded row stride
    const int rowsP = TY + 4, rowsR = TY + 2;
    const int PS = nx * ny;                        // plane stride (elements)
    const size_t N = (size_t)PS * nz;
    const int j0 = tile * TY;
    const int ty_own = min(TY, ny - j0);

    double2* slotR = reinterpret_cast<double2*>(smem_raw);                 // [NS][rowsP][W]
    double2* slotP = slotR + NS * rowsP * W;                                // [NS][rowsP][W]
    double2* rn = slotP + NS * rowsP * W;                                   // [3][rowsR][W]
    uint64_t* bars = reinterpret_cast<uint64_t*>(rn + 3 * rowsR * W);
    double* scratch = reinterpret_cast<double*>(bars + NS);
    __shared__ Scalars sh_sc;

    if (threadIdx.x == 0) sh_sc = pass_scalars(a, rhs, tile);
    __syncthreads();
    const Scalars sc = sh_sc;
    if (!sc.active) return;
    const double2 alpha = sc.alpha, beta = sc.beta;
    const bool first = (a.k == 0);
    const double shift = a.shift[rhs];
    const int kin = a.k & 1, kout = kin ^ 1;
    const double2* __restrict__ Rin = a.R[kin] + (size_t)rhs * N;
    const double2* __restrict__ Pin = a.Pv[kin] + (size_t)rhs * N;
    double2* __restrict__ Rout = a.R[kout] + (size_t)rhs * N;
    double2* __restrict__ Pout = a.Pv[kout] + (size_t)rhs * N;
    double2* __restrict__ Xf = FULLX ? a.X + (size_t)rhs * N : nullptr;
    const double* __restrict__ mu = a.mu;
    const double cx = a.op.cx, cy = a.op.cy, cz = a.op.cz, robin = a.op.robin;

    // slot rows holding in-domain grid rows: [rlo, rhi); grid row of slot row r = j0 - 2 + r
    const int rlo = max(0, 2 - j0), rhi = min(rowsP, ny - j0 + 2);
    const uint32_t row_bytes = (uint32_t)(nx * sizeof(double2));
    const uint32_t plane_bytes = (uint32_t)(rhi - rlo) * row_bytes;
    const int tile_off = (j0 - 2 + rlo) * nx;      // first in-domain element of a plane tile

    for (int idx = threadIdx.x; idx < NS * rowsP * W; idx += blockDim.x) {
        slotR[idx] = cmk(0, 0);
        slotP[idx] = cmk(0, 0);
    }
    for (int idx = threadIdx.x; idx < 3 * rowsR * W; idx += blockDim.x) rn[idx] = cmk(0, 0);
    if (threadIdx.x == 0) {
        for (int s = 0; s < NS; ++s) mbar_init(&bars[s], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int PD = NS - 3;
    auto issue = [&](int z) {       // warp 0: lane 0 arms the barrier, lanes copy one row each
        const int s = z % NS;
        if (lane == 0) {
            fence_proxy_async();
            mbar_expect_tx(&bars[s], first ? plane_bytes : 2 * plane_bytes);
        }
        __syncwarp();
        const int gz = z * PS + (j0 - 2) * nx;
        for (int r = rlo + lane; r < rhi; r += 32) {
            const int o = (s * rowsP + r) * W + 1;
            bulk_g2s(slotR + o, Rin + gz + r * nx, row_bytes, &bars[s]);
            if (!first) bulk_g2s(slotP + o, Pin + gz + r * nx, row_bytes, &bars[s]);
        }
    };
    auto prefetch_l2 = [&](int z) {   // one contiguous block per vector
        const int gz = z * PS + tile_off;
        asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Rin + gz), "r"(plane_bytes) : "memory");
        if (!first)
            asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(Pin + gz), "r"(plane_bytes) : "memory");
    };
    if (warp == 0)
        for (int z = 0; z < PD && z < nz; ++z) issue(z);
    if (warp == 1 && lane == 0)
        for (int z = PD; z < PD + LPD && z < nz; ++z) prefetch_l2(z);

    // ---- per-thread geometry, fixed for the whole march
    const bool act = threadIdx.x < nx * RPT;
    const int ci = act ? threadIdx.x % nx : 0;
    const int rl = act ? threadIdx.x / nx : RPT;
    int p1s[MAXR], p1g[MAXR];        // phase 1: slot offset, global offset in plane (-1: not owned)
    bool p1v[MAXR];
    int p3s[MAXR], p3g[MAXR];        // phase 3 (owned rows): rn offset, global offset
    bool p3v[MAXR];
    int p2s[MAXR], p2g[MAXR];        // phase C: slot offset, mu offset in plane
    bool p2v[MAXR], p2o[MAXR];
#pragma unroll
    for (int m = 0; m < MAXR; ++m) {
        // phase 1 covers TY+4 rows: give its extra rows to the threads with fewer phase-C rows
        const int r1 = rlo + (act ? (rl + RPT / 2) % RPT : RPT) + m * RPT;
        p1v[m] = act && r1 < rhi;
        p1s[m] = r1 * W + ci + 1;
        p1g[m] = (r1 - 2 >= 0 && r1 - 2 < ty_own) ? (j0 + r1 - 2) * nx + ci : -1;
        const int jr = rl + m * RPT;
        p3v[m] = act && jr < ty_own;
        p3s[m] = (jr + 1) * W + ci + 1;
        p3g[m] = (j0 + jr) * nx + ci;
        const int r2 = 1 + rl + m * RPT;
        p2v[m] = act && r2 <= TY + 2 && r2 >= rlo && r2 < rhi;
        p2s[m] = r2 * W + ci + 1;
        p2g[m] = (j0 - 2 + r2) * nx + ci;
        p2o[m] = (r2 - 2 >= 0 && r2 - 2 < ty_own);
    }
    const double dbase = 2.0 * cx + 2.0 * cy;
    const int32_t* soff = a.samp_off + tile;

    double acc[kNumPartials];
#pragma unroll
    for (int q = 0; q < kNumPartials; ++q) acc[q] = 0;

    for (int f = 0; f < nz + 3; ++f) {
        if (warp == 0 && f + PD < nz) issue(f + PD);
        if (warp == 1 && lane == 0 && f + PD + LPD < nz) prefetch_l2(f + PD + LPD);
        const int g = f - 1, t = f - 3;
        const bool do3 = t >= 0 && t < nz, do2 = g >= 0 && g < nz;
        double mu3[MAXR], mu2[MAXR];
#pragma unroll
        for (int m = 0; m < MAXR; ++m) {
            mu3[m] = (do3 && p3v[m]) ? mu[t * PS + p3g[m]] : 0.0;
            mu2[m] = (do2 && p2v[m]) ? mu[g * PS + p2g[m]] : 0.0;
        }
        // ---- B1: phase 1, plane f
        if (f < nz) {
            const int s = f % NS;
            mbar_wait(&bars[s], (uint32_t)((f / NS) & 1));
            double2* sp = slotP + s * rowsP * W;
            const double2* sr = slotR + s * rowsP * W;
            const int fo = f * PS;
#pragma unroll
            for (int m = 0; m < MAXR; ++m) {
                if (!p1v[m]) continue;
                const double2 rv = sr[p1s[m]];
                const double2 pv = first ? rv : cfma(beta, sp[p1s[m]], rv);
                sp[p1s[m]] = pv;
                if (p1g[m] >= 0) {
                    Pout[fo + p1g[m]] = pv;
                    if (FULLX) Xf[fo + p1g[m]] = cfma(alpha, pv, Xf[fo + p1g[m]]);
                }
            }
        }
        // ---- B2: phase 3, plane t: A r_{k+1}, reductions, write r_{k+1}
        if (do3) {
            const double2* rc = rn + (t % 3) * rowsR * W;
            const double2* rd = rn + ((t + 2) % 3) * rowsR * W;
            const double2* ru = rn + ((t + 1) % 3) * rowsR * W;
            const bool edge = (t == 0 || t == nz - 1);
            const double th = edge ? 0.5 : 1.0;
            const double thx = th * cx, thy = th * cy;
            const double dre = th * dbase + cz * (edge ? 1.0 : 2.0) + (edge ? robin : 0.0);
            const double dim = th * shift;
            const double wd = t > 0 ? cz : 0.0, wu = t < nz - 1 ? cz : 0.0;
            const int to = t * PS;
#pragma unroll
            for (int m = 0; m < MAXR; ++m) {
                if (!p3v[m]) continue;
                const int o = p3s[m];
                const double2 r0 = rc[o];
                const double2 sx = cadd(rc[o - 1], rc[o + 1]);
                const double2 sy = cadd(rc[o - W], rc[o + W]);
                const double2 zd = rd[o], zu = ru[o];
                const double dr = fma(th, mu3[m], dre);
                double2 ar;
                ar.x = dr * r0.x - dim * r0.y - thx * sx.x - thy * sy.x - wd * zd.x - wu * zu.x;
                ar.y = dr * r0.y + dim * r0.x - thx * sx.y - thy * sy.y - wd * zd.y - wu * zu.y;
                acc[0] = fma(r0.x, r0.x, fma(-r0.y, r0.y, acc[0]));
                acc[1] = fma(2.0 * r0.x, r0.y, acc[1]);
                acc[2] = fma(r0.x, ar.x, fma(-r0.y, ar.y, acc[2]));
                acc[3] = fma(r0.x, ar.y, fma(r0.y, ar.x, acc[3]));
                acc[8] = fma(r0.x, r0.x, fma(r0.y, r0.y, acc[8]));
                Rout[to + p3g[m]] = r0;
            }
        }
        __syncthreads();
        // ---- C: phase 2, plane g: q = A p_k, r_{k+1} = r_k - alpha q (slot rows 1 .. TY+2)
        if (do2) {
            const int sg = g % NS;
            const double2* pc = slotP + sg * rowsP * W;
            const double2* pd = slotP + ((g + NS - 1) % NS) * rowsP * W;
            const double2* pu = slotP + ((g + 1) % NS) * rowsP * W;
            const double2* rc = slotR + sg * rowsP * W;
            double2* rno = rn + (g % 3) * rowsR * W - W;          // slot row r -> rn row r - 1
            const bool edge = (g == 0 || g == nz - 1);
            const double th = edge ? 0.5 : 1.0;
            const double thx = th * cx, thy = th * cy;
            const double dre = th * dbase + cz * (edge ? 1.0 : 2.0) + (edge ? robin : 0.0);
            const double dim = th * shift;
            const double wd = g > 0 ? cz : 0.0, wu = g < nz - 1 ? cz : 0.0;
#pragma unroll
            for (int m = 0; m < MAXR; ++m) {
                if (!p2v[m]) continue;
                const int o = p2s[m];
                const double2 p0 = pc[o];
                const double2 sx = cadd(pc[o - 1], pc[o + 1]);
                const double2 sy = cadd(pc[o - W], pc[o + W]);
                const double2 zd = pd[o], zu = pu[o];
                const double dr = fma(th, mu2[m], dre);
                double2 q;
                q.x = dr * p0.x - dim * p0.y - thx * sx.x - thy * sy.x - wd * zd.x - wu * zu.x;
                q.y = dr * p0.y + dim * p0.x - thx * sx.y - thy * sy.y - wd * zd.y - wu * zu.y;
                const double2 rnew = csub(rc[o], cmul(alpha, q));
                rno[o] = rnew;
                if (p2o[m]) {
                    acc[4] = fma(rnew.x, q.x, fma(-rnew.y, q.y, acc[4]));
                    acc[5] = fma(rnew.x, q.y, fma(rnew.y, q.x, acc[5]));
                    acc[6] = fma(p0.x, q.x, fma(-p0.y, q.y, acc[6]));
                    acc[7] = fma(p0.x, q.y, fma(p0.y, q.x, acc[7]));
                }
            }
            if (!FULLX && a.nP > 0) {
                const int s0 = soff[g * ntiles], s1 = soff[g * ntiles + 1];
                double2* XP = a.XP + (size_t)rhs * a.nP;
                for (int sidx = s0 + threadIdx.x; sidx < s1; sidx += blockDim.x) {
                    const int rem = a.samp_nodes[sidx] - g * PS;
                    const int jg = rem / nx, i = rem - jg * nx;
                    XP[sidx] = cfma(alpha, pc[(jg - j0 + 2) * W + i + 1], XP[sidx]);
                }
            }
        }
        __syncthreads();
    }
    block_reduce_partials(acc, scratch);
    if (threadIdx.x == 0) {
        double* out = a.part[kout] + ((size_t)rhs * ntiles + tile) * kNumPartials;
        for (int q = 0; q < kNumPartials; ++q) out[q] = acc[q];
    }
}

// (A u)(n) from global memory (reference-style stencil; used by init and dot_apply)
__device__ __forceinline__ double2 apply_point(const OpConst& op, const double* mu, double shift,
                                               const double2* u, int i, int j, int k) {
    const int nx = op.nx, ny = op.ny, nz = op.nz;
    const size_t n = ((size_t)k * ny + j) * nx + i;
    const double2 u0 = u[n];
    double2 lx = cmk(0, 0), ly = cmk(0, 0), lz = cmk(0, 0);
    if (i > 0) lx = cadd(lx, u[n - 1]);
    if (i < nx - 1) lx = cadd(lx, u[n + 1]);
    if (j > 0) ly = cadd(ly, u[n - nx]);
    if (j < ny - 1) ly = cadd(ly, u[n + nx]);
    if (k > 0) lz = cadd(lz, u[n - (size_t)nx * ny]);
    if (k < nz - 1) lz = cadd(lz, u[n + (size_t)nx * ny]);
    const double th = theta_of(k, nz);
    double2 r = cmul(diag_of(op, k, mu[n], shift), u0);
    r = csub(r, cscale(cadd(cscale(lx, op.cx), cscale(ly, op.cy)), th));
    r = csub(r, cscale(lz, op.cz));
    return r;
}

// partials[0]: rho_0 = b^T b, mu_0 = b^T A b, |b|^2 (tile-owned rows, all planes)
__global__ void __launch_bounds__(256) cocg_init_kernel(const PassArgs a) {
    __shared__ double scratch[8 * kNumPartials];
    const int tile = blockIdx.x, rhs = blockIdx.y;
    const int nx = a.op.nx, ny = a.op.ny, nz = a.op.nz;
    const size_t N = (size_t)nx * ny * nz;
    const int j0 = tile * a.tl.TY, ty_own = min(a.tl.TY, ny - j0);
    const double2* b = a.R[0] + (size_t)rhs * N;
    const double shift = a.shift[rhs];
    double acc[kNumPartials];
    for (int i = 0; i < kNumPartials; ++i) acc[i] = 0;
    const int per_plane = ty_own * nx;
    for (int idx = threadIdx.x; idx < per_plane * nz; idx += blockDim.x) {
        const int k = idx / per_plane, rem = idx - k * per_plane;
        const int j = j0 + rem / nx, i = rem % nx;
        const double2 r0 = b[((size_t)k * ny + j) * nx + i];
        if (r0.x == 0.0 && r0.y == 0.0) continue;
        const double2 ar = apply_point(a.op, a.mu, shift, b, i, j, k);
        acc[0] = fma(r0.x, r0.x, fma(-r0.y, r0.y, acc[0]));
        acc[1] = fma(2.0 * r0.x, r0.y, acc[1]);
        acc[2] = fma(r0.x, ar.x, fma(-r0.y, ar.y, acc[2]));
        acc[3] = fma(r0.x, ar.y, fma(r0.y, ar.x, acc[3]));
        acc[8] = fma(r0.x, r0.x, fma(r0.y, r0.y, acc[8]));
    }
    block_reduce_partials(acc, scratch);
    if (threadIdx.x == 0) {
        // slot tile of z chunk 0 carries the sums; the slots of the other z chunks are zero
        double* out = a.part[0] + ((size_t)rhs * a.tl.ntiles * a.nzch_tot + tile) * kNumPartials;
        for (int i = 0; i < kNumPartials; ++i) out[i] = acc[i];
        for (int zc = 1; zc < a.nzch_tot; ++zc)
            for (int i = 0; i < kNumPartials; ++i) out[(size_t)zc * a.tl.ntiles * kNumPartials + i] = 0.0;
    }
    if (threadIdx.x == 0 && tile == 0) {
        RhsState s{};
        a.st[1][rhs] = s;     // pass 0 reads st[1]: not done
    }
}

__global__ void apply_kernel(OpConst op, const double* mu, const double* shift, const double2* u,
                             double2* Au, int nb) {
    const size_t N = (size_t)op.nx * op.ny * op.nz;
    const int rhs = blockIdx.y;
    for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N;
         n += (size_t)gridDim.x * blockDim.x) {
        const int i = n % op.nx, j = (n / op.nx) % op.ny, k = n / ((size_t)op.nx * op.ny);
        Au[(size_t)rhs * N + n] = apply_point(op, mu, shift[rhs], u + (size_t)rhs * N, i, j, k);
    }
}

__global__ void count_active_kernel(const RhsState* st, int nb, int* out, int32_t* act) {
    // one block: ordered compaction of the not-done RHS (block-wide exclusive scan per chunk)
    __shared__ int wsum[32];
    __shared__ int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c0 = 0; c0 < nb; c0 += blockDim.x) {
        const int r = c0 + threadIdx.x;
        const int a = (r < nb && !st[r].done) ? 1 : 0;
        int x = a;                                            // inclusive warp scan
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[warp] = x;
        __syncthreads();
        if (warp == 0) {
            int w = lane < nw ? wsum[lane] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, w, o);
                if (lane >= o) w += y;
            }
            if (lane < nw) wsum[lane] = w;                    // inclusive warp totals
        }
        __syncthreads();
        const int pos = base + (warp > 0 ? wsum[warp - 1] : 0) + x - a;
        if (a && act) act[pos] = r;
        __syncthreads();
        if (threadIdx.x == 0) base += wsum[nw - 1];
        __syncthreads();
    }
    if (act)   // entries past the count: no RHS (a pass launched with an older, larger count skips them)
        for (int y = base + threadIdx.x; y < nb; y += blockDim.x) act[y] = -1;
    if (threadIdx.x == 0) *out = base;
}

__global__ void scatter_rhs_kernel(double2* R0, size_t N, long long rg0, int ncols, const int32_t* nodes,
                                   int nnodes, const double* coeff, const double* scale) {
    const int r = blockIdx.x;
    const int c = (int)((rg0 + r) % ncols);
    for (int a = threadIdx.x; a < nnodes; a += blockDim.x) {
        const double w = coeff ? coeff[(size_t)a * ncols + c] : (a == c ? 1.0 : 0.0);
        if (w != 0.0) R0[(size_t)r * N + nodes[a]] = cmk(w * scale[a], 0.0);
    }
}

__global__ void fill_shift_kernel(double* shift, int nb, long long rg0, int ncols, const double* w) {
    for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < nb; r += gridDim.x * blockDim.x)
        shift[r] = w[(rg0 + r) / ncols];
}

}  // namespace

static CocgTiling ring_tiling(int nx, int ny, int nz, int prefetch, size_t max_smem, int max_threads) {
    CocgTiling t;
    t.kind = 0;
    const size_t budget = max_smem ? max_smem : 225 * 1024;
    const int NS = prefetch + 3;
    const int RPT = std::max(1, (max_threads > 0 ? std::min(max_threads, 512) : 512) / nx);
    const size_t row = (size_t)(nx + 2) * sizeof(double2);
    auto smem_of = [&](int TY) {
        return (size_t)NS * 2 * (TY + 4) * row + 3 * (TY + 2) * row + NS * 8 + (16 * kNumPartials + 8) * 8 + 256;
    };
    int best = 0;
    // phase loops cover at most MAXR = 4 rows per thread; phase 1 has TY + 4 rows
    for (int ty = 1; ty <= ny && ty + 4 <= 4 * RPT; ++ty)
        if (smem_of(ty) <= budget) best = ty;
    if (best <= 0) throw Error(DOT_ERR_ARG, "grid rows too long for the shared-memory plane ring (nx too large)");
    const int ntiles = (ny + best - 1) / best;
    t.TY = (ny + ntiles - 1) / ntiles;      // balanced tiles
    t.ntiles = (ny + t.TY - 1) / t.TY;
    t.nslots = NS;
    t.rpt = RPT;
    t.threads = (nx * RPT + 31) / 32 * 32;
    t.smem = smem_of(t.TY);
    return t;
}

// z-register pass tiling (cocg_z.cu): a thread owns `rows` slot rows of one column
// of the TY + 4 slot rows.  Options in order of preference:
//   D: 2 rows per thread, <= 512 threads, one CTA per SM
//   B: 1 row per thread, <= 768 threads, one CTA per SM (78 registers, no spills)
//   C: 1 row, <= 1024 threads (64 registers)     A: 1 row, <= 512 threads, two CTAs per SM
//   E: 3 rows, <= 384 threads                     F: 4 rows, <= 256 threads
//   G: 2 rows, <= 256 threads, two CTAs per SM
// The first option whose tile height reaches 4 rows wins, else the one with the largest TY.
// DOT_COCG_ZOPT=A..F forces one option (E and F are only tried when forced).
static bool z_tiling(int nx, int ny, int nz, int prefetch, int want_ty, CocgTiling& out) {
    const int NS = prefetch + 2;
    const size_t sm_cta = 227 * 1024, sm_sm = 228 * 1024 - 2048;
    struct Opt { char name; int rows, maxt, minb; };
    const Opt opts[7] = {{'D', 2, 512, 1}, {'B', 1, 768, 1}, {'C', 1, 1024, 1}, {'A', 1, 512, 2},
                         {'E', 3, 384, 1}, {'F', 4, 256, 1}, {'G', 2, 256, 2}};
    const char* eO = std::getenv("DOT_COCG_ZOPT");
    CocgTiling best;
    bool found = false;
    for (const Opt& o : opts) {
        if (eO ? eO[0] != o.name : (o.name == 'E' || o.name == 'F' || o.name == 'G')) continue;
        int ty = 0;
        for (int c = 1; c <= ny; ++c) {
            const int thr = ((c + 4 + o.rows - 1) / o.rows * nx + 31) / 32 * 32;
            const size_t sm = zpass_smem(nx, c, NS, nz);
            if (thr > o.maxt || sm > sm_cta || (size_t)o.minb * (sm + 1024) > sm_sm) break;
            ty = c;
            if (want_ty > 0 && c == want_ty) break;
        }
        if (want_ty > 0 && ty != want_ty) continue;
        if (ty <= 0) continue;
        const int ntiles = (ny + ty - 1) / ty;
        CocgTiling t;
        t.kind = 1;
        t.minb = o.minb;
        t.zrows = o.rows;
        t.TY = (ny + ntiles - 1) / ntiles;
        t.ntiles = (ny + t.TY - 1) / t.TY;
        t.nslots = NS;
        t.threads = ((t.TY + 4 + o.rows - 1) / o.rows * nx + 31) / 32 * 32;
        t.smem = zpass_smem(nx, t.TY, NS, nz);
        if (!found || (best.TY < 4 && t.TY > best.TY)) {
            best = t;
            found = true;
        }
        if (best.TY >= 4 || want_ty > 0) break;
    }
    if (found) out = best;
    return found;
}

CocgTiling cocg_tiling(int nx, int ny, int nz, int prefetch, size_t max_smem, int max_threads, int kind,
                       int want_ty) {
    if (kind != 0) {
        CocgTiling t;
        if (z_tiling(nx, ny, nz, std::max(1, std::min(prefetch, 3)), want_ty, t)) return t;
        if (kind == 1 && want_ty > 0) throw Error(DOT_ERR_ARG, "requested z-pass tile height does not fit");
    }
    return ring_tiling(nx, ny, nz, std::max(1, prefetch - (kind != 0 ? 1 : 0)), max_smem, max_threads);
}

void launch_cocg_init(const PassArgs& a, int nb, cudaStream_t s) {
    dim3 grid(a.tl.ntiles, nb);
    cocg_init_kernel<<<grid, 256, 0, s>>>(a);
    DOT_CUDA_TRY(cudaGetLastError());
}

// Compile-time geometries of the BASELINE.json grids (nx, TY, slots, rows per sweep);
// any other geometry runs the run-time-parameter instance <.., 0, 0, 0, 0>.
#define DOT_COCG_GEOMS(X) X(16, 16, 4, 32) X(32, 32, 4, 16) X(64, 16, 4, 8) X(96, 9, 4, 5) X(128, 6, 4, 4)

template <bool FX>
static void launch_pass_impl(const PassArgs& a, int nb, cudaStream_t s) {
    using K = void (*)(const PassArgs);
    K k = cocg_pass_kernel<FX, 0, 0, 0, 0>;
#define DOT_PICK(GX, GT, GS, GR) \
    if (a.op.nx == GX && a.tl.TY == GT && a.tl.nslots == GS && a.tl.rpt == GR) k = cocg_pass_kernel<FX, GX, GT, GS, GR>;
    DOT_COCG_GEOMS(DOT_PICK)
#undef DOT_PICK
    ensure_smem(k, a.tl.smem);
    dim3 grid(a.tl.ntiles, nb);
    launch_clustered(k, grid, a.tl.threads, a.tl.smem, s, a.tl.cluster, a);
}

void launch_cocg_pass(const PassArgs& a, int nb, cudaStream_t s) {
    if (a.tl.kind == 1) {
        launch_cocg_zpass(a, nb, s);
        return;
    }
    if (a.X) launch_pass_impl<true>(a, nb, s);
    else launch_pass_impl<false>(a, nb, s);
}

void launch_count_active(const RhsState* st, int nb, int* d_count, cudaStream_t s, int32_t* act) {
    count_active_kernel<<<1, 256, 0, s>>>(st, nb, d_count, act);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_apply(const OpConst& op, const double* mu, const double* shift, const double2* u,
                  double2* Au, int nb, cudaStream_t s) {
    const size_t N = (size_t)op.nx * op.ny * op.nz;
    dim3 grid((unsigned)std::min<size_t>((N + 255) / 256, 4096), nb);
    apply_kernel<<<grid, 256, 0, s>>>(op, mu, shift, u, Au, nb);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_scatter_rhs(double2* R0, size_t N, int nb, long long rg0, int ncols, const int32_t* nodes,
                        int nnodes, const double* coeff, const double* scale, cudaStream_t s) {
    scatter_rhs_kernel<<<nb, 256, 0, s>>>(R0, N, rg0, ncols, nodes, nnodes, coeff, scale);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_fill_shift(double* shift, int nb, long long rg0, int ncols, const double* omega_over_nu,
                       cudaStream_t s) {
    fill_shift_kernel<<<(nb + 255) / 256, 256, 0, s>>>(shift, nb, rg0, ncols, omega_over_nu);
    DOT_CUDA_TRY(cudaGetLastError());
}

}  // namespace dot
