// Fused single-pass COCG iteration, z-march with register-resident z-neighbours
// ("COCG pass tiling"; PAPER.md L966 solves of Eq. (2.1)).
//
// Same recurrences as cocg_pass_kernel (cocg.cu): pass k forms
//   p_k = r_k + beta_k p_{k-1},  q = A p_k,  r_{k+1} = r_k - alpha_k q
// with rho, mu = r^T A r, nu = r^T q and sigma_direct = p^T q reduced in the same
// sweep; 64 B of HBM traffic per point and iteration (read r_k, p_{k-1}; write
// p_k, r_{k+1}).
//
// Mapping: a CTA owns TY full x-rows (grid rows j0 .. j0+TY-1) of one RHS and
// marches the nz planes.  One thread per (x, slot row) of the TY+4 slot rows:
//   slot rows 2 .. TY+1   own rows:  phase 1 (p_k), 2 (q, r_{k+1}), 3 (A r_{k+1})
//   slot rows 1, TY+2     y-halo 1:  phases 1, 2   (r_{k+1} feeds the own rows' stencil)
//   slot rows 0, TY+3     y-halo 2:  phase 1       (p_k feeds the halo-1 stencil)
// Each thread keeps its own column's p_k and r_{k+1} of the two previous planes
// in registers, so the z-neighbours of both stencils never touch shared memory;
// only the 4 in-plane neighbours are read from shared memory.
//
// Per plane f (one __syncthreads per plane):
//   producer  one cp.async.bulk per vector: the TY+4 contiguous rows of r_k and
//             p_{k-1} of plane f+PD into ring slot (f+PD) % NS   (NS = PD + 2)
//   phase 1   plane f:   p_k = r_k + beta p_{k-1}, written in place into the slot
//   phase 2   plane f-1: q = A p_k, r_{k+1} = r_k - alpha q -> Rbuf[(f-1) % 3]
//   phase 3   plane f-2: A r_{k+1}, reductions, store r_{k+1}
#include "kernels.h"

namespace dot {

namespace {

__device__ __forceinline__ uint32_t smem_u32z(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double warp_sum_z(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct ZScalars {
    double2 alpha, beta;
    int active;
};

// Scalar recurrences of pass k for one RHS, computed by warp 0 (lanes split the
// tiles, fixed-order butterfly reduction: identical in every CTA of the RHS).
__device__ void zpass_scalars(const PassArgs& a, int rhs, int tile, ZScalars* out) {
    const int lane = threadIdx.x & 31;
    const int ntiles = a.tl.ntiles * a.nzch_tot;      // partial slots per RHS (tiles x global z chunks)
    const double* pp = a.part[a.k & 1] + (size_t)rhs * ntiles * kNumPartials;
    double s[kNumPartials];
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) s[i] = 0.0;
    for (int t = lane; t < ntiles; t += 32)
#pragma unroll
        for (int i = 0; i < kNumPartials; ++i) s[i] += pp[t * kNumPartials + i];
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) s[i] = warp_sum_z(s[i]);
    if (lane != 0) return;
    const RhsState prev = a.st[(a.k + 1) & 1][rhs];
    RhsState cur = prev;
    ZScalars sc;
    sc.alpha = cmk(0, 0);
    sc.beta = cmk(0, 0);
    sc.active = 0;
    if (!prev.done) {
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
        if (!(nrm2 > a.tol2 * cur.bnorm2)) {            // converged (also b = 0)
            cur.done = 1;
            cur.iters = a.k;
        } else if (a.k >= a.max_iter) {
            cur.done = 1;
            cur.iters = a.k;
            cur.flag = DOT_ERR_NOCONV;
        } else if (!isfinite(alpha.x) || !isfinite(alpha.y) || !isfinite(beta.x) || !isfinite(beta.y)) {
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
    if (tile == 0) {
        a.st[a.k & 1][rhs] = cur;
        // a finished RHS may drop out of later launches (active list): freeze both copies
        if (cur.done) a.st[(a.k + 1) & 1][rhs] = cur;
    }
    *out = sc;
}

// Plane coefficients of row n of A at plane k (R1-R3):
//   theta [cx(2u - uW - uE) + cy(2u - uS - uN) + (mu + i shift) u] + cz(nzn u - uD - uU) + robin u
struct PlaneCoef {
    double thx, thy, th, dre, dim, wd, wu;
};
__device__ __forceinline__ PlaneCoef plane_coef(const OpConst& op, int k, double shift) {
    PlaneCoef c;
    const bool edge = (k == 0 || k == op.nz - 1);
    c.th = edge ? 0.5 : 1.0;
    c.thx = c.th * op.cx;
    c.thy = c.th * op.cy;
    c.dre = c.th * (2.0 * op.cx + 2.0 * op.cy) + op.cz * (edge ? 1.0 : 2.0) + (edge ? op.robin : 0.0);
    c.dim = c.th * shift;
    c.wd = k > 0 ? op.cz : 0.0;
    c.wu = k < op.nz - 1 ? op.cz : 0.0;
    return c;
}

__device__ __forceinline__ double2 stencil(const PlaneCoef& c, double mu, double2 u0, double2 sx, double2 sy,
                                           double2 zd, double2 zu) {
    const double dr = fma(c.th, mu, c.dre);
    double2 r;
    r.x = dr * u0.x - c.dim * u0.y - c.thx * sx.x - c.thy * sy.x - c.wd * zd.x - c.wu * zu.x;
    r.y = dr * u0.y + c.dim * u0.x - c.thx * sx.y - c.thy * sy.y - c.wd * zd.y - c.wu * zu.y;
    return r;
}

template <int I>
struct IC {
    static constexpr int v = I;
};

// Interior-plane stencil (theta = 1, both z-neighbours present): coefficients
// straight from the kernel-parameter constant bank, no registers held.
__device__ __forceinline__ double2 stencil_int(const OpConst& op, double shift, double mu, double2 u0, double2 sx,
                                               double2 sy, double2 zs) {
    const double dr = op.dint + mu;
    double2 r;
    r.x = dr * u0.x - shift * u0.y - op.cx * sx.x - op.cy * sy.x - op.cz * zs.x;
    r.y = dr * u0.y + shift * u0.x - op.cx * sx.y - op.cy * sy.y - op.cz * zs.y;
    return r;
}

// Slot layout (per ring slot): r [rowsP*nx] double2 | p [rowsP*nx] double2 | mu [rowsP*nx] double
// (mu rides along in the same bulk-copy group when MUT; else it is loaded per thread).
// RPT: slot rows per thread (a thread owns rows RPT*m .. RPT*m + RPT - 1 of one column; the
// y-neighbours inside its strip come from registers).
template <bool FULLX, int MAXT, int MINB, int NS, bool MUT, int RPT, bool ZC>
__global__ void __launch_bounds__(MAXT, MINB) cocg_zpass_kernel(const __grid_constant__ PassArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int PD = NS - 2;                          // TMA planes in flight
    const int ntiles = a.tl.ntiles;
    const int tile = blockIdx.x % ntiles, zc = a.zc0 + blockIdx.x / ntiles;
    const int rhs = a.act ? a.act[blockIdx.y] : blockIdx.y;       // active-list compaction (tail passes)
    if (rhs < 0) return;                                           // slot past the active count
    const int nx = a.op.nx, ny = a.op.ny, nz = a.op.nz;
    const int TY = a.tl.TY;
    // z chunk [z0, z1) of this CTA; phase 1 runs on [a1, b1), phase 2 on [a2, b2)
    // (two / one halo planes recomputed on each side)
    // (ZC = false: one chunk, the whole z range -- the bounds fold to constants)
    const int z0 = ZC ? zc * a.zlen : 0, z1 = ZC ? min(nz, z0 + a.zlen) : nz;
    const int a1 = ZC ? max(z0 - 2, 0) : 0, b1 = ZC ? min(z1 + 2, nz) : nz;
    const int a2 = ZC ? max(z0 - 1, 0) : 0, b2 = ZC ? min(z1 + 1, nz) : nz;
    const int fend = ZC ? min(b1, z1) + 2 : nz + 2;
    const int rowsP = TY + 4, rowsR = TY + 2;
    const int PS = nx * ny;
    const size_t N = (size_t)PS * nz;
    const int j0 = tile * TY;
    const int slotE = rowsP * nx;                       // double2 elements of one vector in a slot
    const int slotW = 2 * slotE + (MUT ? (slotE + 1) / 2 : 0);   // slot stride in double2
    const int rbE = rowsR * nx;

    double2* slots = reinterpret_cast<double2*>(smem_raw);          // [NS][slotW]
    double2* rbuf = slots + (size_t)NS * slotW;                     // [3][rowsR*nx]
    uint64_t* bars = reinterpret_cast<uint64_t*>(rbuf + 3 * rbE);
    double* scratch = reinterpret_cast<double*>(bars + NS);         // [32][kNumPartials]
    int2* s_samp = reinterpret_cast<int2*>(scratch + 32 * kNumPartials);   // [nz] sample ranges
    __shared__ ZScalars sh_sc;

    if (threadIdx.x < 32) zpass_scalars(a, rhs, blockIdx.x, &sh_sc);
    {   // rows outside the domain (edge tiles only) must read as zero (Dirichlet y faces):
        // the p rows of every ring slot outside [rlo, rhi) and the Rbuf rows outside
        // [rlo - 1, rhi - 1); nothing else is read before it is written
        const int rlo_ = max(0, 2 - j0), rhi_ = min(TY + 4, ny - j0 + 2);
        const int nlo = rlo_ * nx, nhi = (TY + 4 - rhi_) * nx;
        if (nlo + nhi > 0) {
            const int per = nlo + nhi;
            for (int i = threadIdx.x; i < NS * per; i += blockDim.x) {
                const int q = i / per, e = i - q * per;
                const int el = e < nlo ? e : rhi_ * nx + (e - nlo);
                slots[(size_t)q * slotW + slotE + el] = cmk(0, 0);
            }
            const int blo = max(0, rlo_ - 1) * nx, bhi_r = max(0, rhi_ - 1);
            const int bper = blo + (TY + 2 - min(TY + 2, bhi_r)) * nx;
            for (int i = threadIdx.x; i < 3 * bper; i += blockDim.x) {
                const int q = i / bper, e = i - q * bper;
                const int el = e < blo ? e : min(TY + 2, bhi_r) * nx + (e - blo);
                rbuf[(size_t)q * rbE + el] = cmk(0, 0);
            }
        }
        if (!FULLX && a.nP > 0)
            for (int g = threadIdx.x; g < nz; g += blockDim.x)
                s_samp[g] = make_int2(a.samp_off[g * ntiles + tile], a.samp_off[g * ntiles + tile + 1]);
    }
    if (threadIdx.x == 0) {
        for (int q = 0; q < NS; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32z(&bars[q])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (!sh_sc.active) return;
    const bool first = (a.k == 0);
    const double shift = a.shift[rhs];
    const int kin = a.k & 1, kout = kin ^ 1;
    const double2* __restrict__ Rin = a.R[kin] + (size_t)rhs * N;
    const double2* __restrict__ Pin = a.Pv[kin] + (size_t)rhs * N;

    // in-domain slot rows [rlo, rhi); grid row of slot row r is j0 - 2 + r
    const int rlo = max(0, 2 - j0), rhi = min(rowsP, ny - j0 + 2);
    const uint32_t tile_bytes = (uint32_t)((rhi - rlo) * nx * sizeof(double2));
    const uint32_t mu_bytes = tile_bytes / 2;
    const uint32_t tx_bytes = (first ? tile_bytes : 2 * tile_bytes) + (MUT ? mu_bytes : 0);
    const int tile_off = (j0 - 2 + rlo) * nx;
    const uint32_t slot0 = smem_u32z(slots + rlo * nx);             // r rows of slot 0
    const uint32_t slot_stride = (uint32_t)(slotW * sizeof(double2));
    const uint32_t pvec_off = (uint32_t)(slotE * sizeof(double2));
    // mu rows land at slot + 2 slotE double2 + rlo*nx doubles (dR already includes rlo*nx double2)
    const uint32_t mu_off = (uint32_t)(2 * slotE * sizeof(double2)) - (uint32_t)(rlo * nx * 8);
    const uint32_t bar0 = smem_u32z(bars);

    auto issue = [&](int z, int sl) {      // one thread: bulk copies of contiguous rows
        const uint32_t dR = slot0 + sl * slot_stride, bar = bar0 + 8 * sl;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx_bytes) : "memory");
        const size_t g = (size_t)z * PS + tile_off;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dR),
            "l"(Rin + g), "r"(tile_bytes), "r"(bar)
            : "memory");
        if (!first)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dR + pvec_off),
                "l"(Pin + g), "r"(tile_bytes), "r"(bar)
                : "memory");
        if (MUT)
            asm volatile(
                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                    dR + mu_off),
                "l"(a.mu + g), "r"(mu_bytes), "r"(bar)
                : "memory");
    };
    if (threadIdx.x == 0)
        for (int z = a1; z < a1 + PD && z < b1; ++z) issue(z, z - a1);

    // ---- per-thread geometry: rows r0 .. r0 + RPT - 1 of column x
    const int t = threadIdx.x;
    const int m = t / nx, x = t - m * nx;
    const int r0 = RPT * m;
    bool indom[RPT], own[RPT], ph2[RPT];
    bool any_in = false, any2 = false, any_own = false;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        const int r = r0 + j;
        indom[j] = r < rowsP && r >= rlo && r < rhi;
        own[j] = indom[j] && r >= 2 && r < TY + 2;
        ph2[j] = own[j] || (indom[j] && (r == 1 || r == TY + 2));
        any_in |= indom[j];
        any2 |= ph2[j];
        any_own |= own[j];
    }
    bool all_in = true, all2 = true, all_own = true;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        all_in &= indom[j];
        all2 &= ph2[j];
        all_own &= own[j];
    }
    const int o = r0 * nx + x;                         // slot element of row 0
    const int o3 = o - nx;                             // Rbuf element of row 0
    const int go = (j0 - 2 + r0) * nx + x;             // plane offset of row 0 (may be outside; unused then)
    const bool hasW = x > 0, hasE = x < nx - 1;
    // running per-thread global pointers (advance one plane per step)
    double2* pP = a.Pv[kout] + (size_t)rhs * N + go + (ptrdiff_t)a1 * PS;        // p_k at plane f
    double2* pR = a.R[kout] + (size_t)rhs * N + go + (ptrdiff_t)(a1 - 2) * PS;   // r_{k+1} at plane f - 2
    double2* pX = FULLX ? a.X + (size_t)rhs * N + go + (ptrdiff_t)a1 * PS : nullptr;
    const double* pMu = a.mu + go;                     // used when !MUT

    double acc[kNumPartials];
#pragma unroll
    for (int q = 0; q < kNumPartials; ++q) acc[q] = 0.0;

    const double2 z2 = cmk(0, 0);
    double2 Pq[RPT][3], RN[RPT][3];    // p_k, r_{k+1} at planes == index mod 3 (own column)
    double MU[RPT][3], mu_carry[RPT];  // mu (register pipeline only when !MUT); mu of plane f - 2
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
#pragma unroll
        for (int q = 0; q < 3; ++q) {
            Pq[j][q] = z2;
            RN[j][q] = z2;
            MU[j][q] = 0.0;
        }
        mu_carry[j] = 0.0;
    }
    int sl = 0;                        // ring slot of plane f
    uint32_t par = 0;                  // mbarrier parity of plane f
    int sl_prev = NS - 1;              // ring slot of plane f - 1
    int sl_iss = PD % NS;              // ring slot of plane f + PD

    auto step = [&](int f, auto IDX) {
        constexpr int i0 = decltype(IDX)::v;           // f % 3
        constexpr int i1 = (i0 + 2) % 3;               // (f - 1) % 3
        constexpr int i2 = (i0 + 1) % 3;               // (f - 2) % 3
        if (threadIdx.x == 0 && f + PD < b1) issue(f + PD, sl_iss);
        const bool ownf = !ZC || (f >= z0 && f < z1);
        if (!MUT && f < b1)
#pragma unroll
            for (int j = 0; j < RPT; ++j)
                if (ph2[j]) MU[j][i0] = pMu[(size_t)f * PS + j * nx];
        // ---- phase 1: plane f
        double2 pf[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) pf[j] = z2;
        if (f < b1) {
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "WAITZ_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAITZ_%=;\n\t}" ::"r"(bar0 + 8 * sl),
                "r"(par)
                : "memory");
            if (any_in) {
                double2* sr = slots + sl * slotW + o;
                const double2 beta = sh_sc.beta;
                auto p1 = [&](auto ALL) {
                    constexpr bool A = decltype(ALL)::v != 0;
#pragma unroll
                    for (int j = 0; j < RPT; ++j) {
                        if (!A && !indom[j]) continue;
                        const double2 rf = sr[j * nx];
                        pf[j] = first ? rf : cfma(beta, sr[slotE + j * nx], rf);
                        sr[slotE + j * nx] = pf[j];
                        if (own[j] && ownf) {
                            pP[j * nx] = pf[j];
                            if (FULLX) pX[j * nx] = cfma(sh_sc.alpha, pf[j], pX[j * nx]);
                        }
                    }
                };
                if (all_in) p1(IC<1>());
                else p1(IC<0>());
            }
        }
        // ---- phase 2: plane g = f - 1
        double2 rng[RPT];
        double mug[RPT];
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            rng[j] = z2;
            mug[j] = 0.0;
        }
        const int g = f - 1;
        if (g >= a2 && g < b2) {
            const bool owng = !ZC || (g >= z0 && g < z1);
            const double2* sr = slots + sl_prev * slotW;
            const double2* sp = sr + slotE;
            if (any2) {
                const bool interior = g > 0 && g < nz - 1;
                const PlaneCoef ce = interior ? PlaneCoef{} : plane_coef(a.op, g, shift);
                const double2 alpha = sh_sc.alpha;
                auto p2 = [&](auto ALL) {
                constexpr bool A = decltype(ALL)::v != 0;
#pragma unroll
                for (int j = 0; j < RPT; ++j) {
                    if (!A && !ph2[j]) continue;
                    const int oj = o + j * nx;
                    const double2 xw = hasW ? sp[oj - 1] : z2;
                    const double2 xe = hasE ? sp[oj + 1] : z2;
                    const double2 ys = j > 0 ? Pq[j > 0 ? j - 1 : 0][i1] : sp[oj - nx];
                    const double2 yn = j < RPT - 1 ? Pq[j < RPT - 1 ? j + 1 : 0][i1] : sp[oj + nx];
                    mug[j] = MUT ? reinterpret_cast<const double*>(sr + 2 * slotE)[oj] : MU[j][i1];
                    const double2 pc = Pq[j][i1];
                    double2 qv;
                    if (interior)
                        qv = stencil_int(a.op, shift, mug[j], pc, cadd(xw, xe), cadd(ys, yn), cadd(Pq[j][i2], pf[j]));
                    else
                        qv = stencil(ce, mug[j], pc, cadd(xw, xe), cadd(ys, yn), Pq[j][i2], pf[j]);
                    rng[j] = csub(sr[oj], cmul(alpha, qv));
                    rbuf[i1 * rbE + o3 + j * nx] = rng[j];
                    if (own[j] && owng) {
                        acc[4] = fma(rng[j].x, qv.x, fma(-rng[j].y, qv.y, acc[4]));
                        acc[5] = fma(rng[j].x, qv.y, fma(rng[j].y, qv.x, acc[5]));
                        acc[6] = fma(pc.x, qv.x, fma(-pc.y, qv.y, acc[6]));
                        acc[7] = fma(pc.x, qv.y, fma(pc.y, qv.x, acc[7]));
                    }
                }
                };
                if (all2) p2(IC<1>());
                else p2(IC<0>());
            }
            if (!FULLX && a.nP > 0 && owng) {
                const int2 sr2 = s_samp[g];
                if (sr2.x < sr2.y) {
                    double2* XP = a.XP + (size_t)rhs * a.nP;
                    for (int si = sr2.x + threadIdx.x; si < sr2.y; si += blockDim.x) {
                        const int rem = a.samp_nodes[si] - g * PS;
                        XP[si] = cfma(sh_sc.alpha, sp[rem - (j0 - 2) * nx], XP[si]);
                    }
                }
            }
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) Pq[j][i0] = pf[j];
        // ---- phase 3: plane tt = f - 2
        const int tt = f - 2;
        if (any_own && tt >= z0 && tt < z1) {
            const double2* rc = rbuf + i2 * rbE + o3;
            const bool interior = tt > 0 && tt < nz - 1;
            const PlaneCoef ce = interior ? PlaneCoef{} : plane_coef(a.op, tt, shift);
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                if (!own[j]) continue;
                const double2 xw = hasW ? rc[j * nx - 1] : z2;
                const double2 xe = hasE ? rc[j * nx + 1] : z2;
                // y-neighbours: own-strip rows from registers (r_{k+1} of plane tt is RN[.][i2])
                const double2 ys = j > 0 ? RN[j > 0 ? j - 1 : 0][i2] : rc[(j - 1) * nx];
                const double2 yn = j < RPT - 1 ? RN[j < RPT - 1 ? j + 1 : 0][i2] : rc[(j + 1) * nx];
                const double2 r0v = RN[j][i2];
                const double mut = MUT ? mu_carry[j] : MU[j][i2];
                double2 ar;
                if (interior)
                    ar = stencil_int(a.op, shift, mut, r0v, cadd(xw, xe), cadd(ys, yn), cadd(RN[j][i0], rng[j]));
                else
                    ar = stencil(ce, mut, r0v, cadd(xw, xe), cadd(ys, yn), RN[j][i0], rng[j]);
                acc[0] = fma(r0v.x, r0v.x, fma(-r0v.y, r0v.y, acc[0]));
                acc[1] = fma(2.0 * r0v.x, r0v.y, acc[1]);
                acc[2] = fma(r0v.x, ar.x, fma(-r0v.y, ar.y, acc[2]));
                acc[3] = fma(r0v.x, ar.y, fma(r0v.y, ar.x, acc[3]));
                acc[8] = fma(r0v.x, r0v.x, fma(r0v.y, r0v.y, acc[8]));
                pR[j * nx] = r0v;
            }
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            RN[j][i1] = rng[j];
            mu_carry[j] = mug[j];
        }
        pP += PS;
        pR += PS;
        if (FULLX) pX += PS;
        sl_prev = sl;
        if (++sl == NS) {
            sl = 0;
            par ^= 1u;
        }
        if (++sl_iss == NS) sl_iss = 0;
        __syncthreads();
    };
    // RN[.][i0] read in phase 3 is r_{k+1}(f-3), written three steps earlier.
#pragma unroll 1
    for (int f = a1; f < fend; f += 3) {
        step(f, IC<0>());
        if (f + 1 < fend) step(f + 1, IC<1>());
        if (f + 2 < fend) step(f + 2, IC<2>());
    }
    // ---- deterministic block reduction of the partials
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = (blockDim.x + 31) >> 5;
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) acc[i] = warp_sum_z(acc[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < kNumPartials; ++i) scratch[warp * kNumPartials + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < kNumPartials) {
        double sum = 0;
        for (int w = 0; w < nw; ++w) sum += scratch[w * kNumPartials + threadIdx.x];
        a.part[kout][((size_t)rhs * ntiles * a.nzch_tot + (size_t)zc * ntiles + tile) * kNumPartials + threadIdx.x] = sum;
    }
}

template <bool FX, int MAXT, int MINB, int NS, int RPT>
void launch_z_ns(const PassArgs& a, int nb, cudaStream_t s) {
    // mu rides in the bulk-copy group when every copy is 16-byte sized and aligned
    const bool mut = (a.op.nx % 2 == 0);
    const bool zc = a.nzch > 1 || a.nzch_tot > 1;
    auto k = mut ? (zc ? cocg_zpass_kernel<FX, MAXT, MINB, NS, true, RPT, true>
                       : cocg_zpass_kernel<FX, MAXT, MINB, NS, true, RPT, false>)
                 : (zc ? cocg_zpass_kernel<FX, MAXT, MINB, NS, false, RPT, true>
                       : cocg_zpass_kernel<FX, MAXT, MINB, NS, false, RPT, false>);
    ensure_smem(k, a.tl.smem);
    dim3 grid(a.tl.ntiles * a.nzch, nb);
    launch_clustered(k, grid, a.tl.threads, a.tl.smem, s, a.nzch == 1 ? a.tl.cluster : 1, a);
}

template <bool FX, int MAXT, int MINB, int RPT>
void launch_z(const PassArgs& a, int nb, cudaStream_t s) {
    switch (a.tl.nslots) {
        case 3: launch_z_ns<FX, MAXT, MINB, 3, RPT>(a, nb, s); break;
        case 4: launch_z_ns<FX, MAXT, MINB, 4, RPT>(a, nb, s); break;
        case 5: launch_z_ns<FX, MAXT, MINB, 5, RPT>(a, nb, s); break;
        default: throw Error(DOT_ERR_ARG, "z pass supports 3..5 ring slots (DOT_COCG_PREFETCH 1..3)");
    }
}

}  // namespace

size_t zpass_smem(int nx, int TY, int NS, int nz) {
    const size_t slotE = (size_t)(TY + 4) * nx;
    const size_t e = (size_t)NS * (2 * slotE + (nx % 2 == 0 ? (slotE + 1) / 2 : 0)) + 3 * (size_t)(TY + 2) * nx;
    return e * sizeof(double2) + NS * 8 + 32 * kNumPartials * 8 + 8 * (size_t)nz + 128;
}

void launch_cocg_zpass(const PassArgs& a, int nb, cudaStream_t s) {
    const int maxt = a.tl.threads;
    if (a.tl.zrows >= 2) {
        if (maxt > 512) throw Error(DOT_ERR_ARG, "z pass with 2..4 rows per thread supports <= 512 threads");
        if (a.tl.zrows == 2 && a.tl.minb >= 2) {
            if (a.X) launch_z<true, 512, 1, 2>(a, nb, s);
            else launch_z<false, 256, 2, 2>(a, nb, s);
        } else if (a.tl.zrows == 2) {
            if (a.X) launch_z<true, 512, 1, 2>(a, nb, s);
            else launch_z<false, 512, 1, 2>(a, nb, s);
        } else if (a.tl.zrows == 3) {
            if (a.X) launch_z<true, 384, 1, 3>(a, nb, s);
            else launch_z<false, 384, 1, 3>(a, nb, s);
        } else {
            if (a.X) launch_z<true, 256, 1, 4>(a, nb, s);
            else launch_z<false, 256, 1, 4>(a, nb, s);
        }
        return;
    }
    if (a.X) {
        if (maxt <= 512) launch_z<true, 512, 1, 1>(a, nb, s);
        else launch_z<true, 1024, 1, 1>(a, nb, s);
        return;
    }
    if (a.tl.minb >= 2) launch_z<false, 512, 2, 1>(a, nb, s);
    else if (maxt <= 512) launch_z<false, 512, 1, 1>(a, nb, s);
    else if (maxt <= 768) launch_z<false, 768, 1, 1>(a, nb, s);
    else launch_z<false, 1024, 1, 1>(a, nb, s);
}

}  // namespace dot
