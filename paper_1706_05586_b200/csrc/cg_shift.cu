// Multi-shift conjugate gradients for all frequencies of the DOT operator at once
// (Eq. (2.1), L183-187 A(p, omega) = A(p, 0) + i omega/nu E,
// and L966 "we solve A(p) z_i = B w_i ... A^T(p) y_j = C v_j").
//
// With Theta = diag(theta) = E (reading R2), the symmetric scaling
//   K~ = Theta^-1/2 A(p, 0) Theta^-1/2,  b~ = Theta^-1/2 b,  x = Theta^-1/2 x~
// turns every frequency into the SAME real SPD matrix plus a scalar shift:
//   Theta^-1/2 A(p, omega) Theta^-1/2 = K~ + i (omega/nu) I.
// Krylov spaces are shift invariant, so one real CG "seed" run on K~ x~ = b~ (b real:
// point sources, point detectors, real W / V combinations) yields the iterates of every
// shifted system by scalar recurrences (shifted CG; the shifted residuals are collinear,
// r_sigma = zeta_sigma r).  The grid sweep moves only the seed's real vectors -- 32 B per
// point and iteration for ALL frequencies, against 64 B per point, iteration and
// frequency for a complex COCG per frequency.  The shifted directions p_sigma and
// solutions x_sigma are pointwise recurrences driven by the seed residual, so they are
// kept only on the sample set P (support S, detectors, sources): the pass writes r_k at
// the samples into a history ring, and a fold kernel applies
//   p_sigma <- zeta_k r_k + beta_sigma p_sigma,   x_sigma <- x_sigma + alpha_sigma p_sigma
// every kHist passes.
//
// Two real seeds share one double2 lane ("pair"): .x and .y are independent CGs with
// their own scalars.  Pass k (single-sweep CG, as the round-1 COCG pass):
//   p_k = r_k + beta_k p_{k-1},  q = K~ p_k,  r_{k+1} = r_k - alpha_k q
// with rho_{k+1} = r^T r, mu_{k+1} = r^T K~ r, nu_{k+1} = r^T q and sigma_direct = p^T q
// reduced in the same sweep; the next pass takes beta = rho_{k+1}/rho_k,
// sigma = mu + 2 beta nu + beta^2 sigma_direct, alpha = rho/sigma.
//
// Mapping (z march): a CTA owns TY full x-rows of one pair and marches the nz planes.
// One thread per (x, RPT consecutive slot rows) of the TY+4 slot rows:
//   slot rows 2 .. TY+1   own rows:  phase 1 (p_k), 2 (q, r_{k+1}), 3 (K~ r_{k+1})
//   slot rows 1, TY+2     y-halo 1:  phases 1, 2
//   slot rows 0, TY+3     y-halo 2:  phase 1
// z-neighbours of both stencils stay in registers; one __syncthreads per plane.
//   producer  one cp.async.bulk per vector: the TY+4 contiguous rows of r_k, p_{k-1}
//             (and mu) of plane f+PD into ring slot (f+PD) % NS   (NS = PD + 2)
//   phase 1   plane f:   p_k = r_k + beta p_{k-1}, written in place into the slot
//   phase 2   plane f-1: q = K~ p_k, r_{k+1} = r_k - alpha q -> Rbuf[(f-1) % 3]; r_k at samples
//   phase 3   plane f-2: K~ r_{k+1}, reductions, store r_{k+1}
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <string>
#include <vector>

#include "kernels.h"

namespace dot {

namespace {

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// theta^-1/2 of plane k: sqrt(2) on the Robin planes (reading R2), 1 inside
__host__ __device__ __forceinline__ double unscale_of(int k, int nz) {
    return (k == 0 || k == nz - 1) ? 1.4142135623730951 : 1.0;
}

// -------------------------------------------------------------- the scaled operator K~
// Row n at plane k of K~ = Theta^-1/2 A(p, 0) Theta^-1/2 (entries A_nm / sqrt(theta_n theta_m)):
//   (dk + mu) u - cx (uW + uE) - cy (uS + uN) - wd uD - wu uU
//   dk = 2 cx + 2 cy + (cz nzn_k + robin_k) / theta_k,  wd = cz / sqrt(theta_k theta_{k-1}), ...
struct PlaneCoef {
    double d, wd, wu;
};
__host__ __device__ __forceinline__ PlaneCoef plane_coef(const OpConst& op, int k) {
    const int nz = op.nz;
    const double th = (k == 0 || k == nz - 1) ? 0.5 : 1.0;
    const double nzn = (k > 0 ? 1.0 : 0.0) + (k < nz - 1 ? 1.0 : 0.0);
    const double rob = (k == 0 || k == nz - 1) ? op.robin : 0.0;
    PlaneCoef c;
    c.d = 2.0 * op.cx + 2.0 * op.cy + (op.cz * nzn + rob) / th;
    c.wd = k > 0 ? op.cz / sqrt(th * ((k - 1 == 0) ? 0.5 : 1.0)) : 0.0;
    c.wu = k < nz - 1 ? op.cz / sqrt(th * ((k + 1 == nz - 1) ? 0.5 : 1.0)) : 0.0;
    return c;
}

// coefficients of the planes 0, 1, nz-2, nz-1 (precomputed on the host, PassArgs::ec)
__device__ __forceinline__ PlaneCoef edge_coef(const PassArgs& a, int k) {
    const int i = k == 0 ? 0 : (k == 1 ? 1 : (k == a.op.nz - 1 ? 3 : 2));
    PlaneCoef c;
    c.d = a.ec[i][0];
    c.wd = a.ec[i][1];
    c.wu = a.ec[i][2];
    return c;
}

// the two real seeds of a pair, componentwise
__device__ __forceinline__ double2 kt_edge(const PlaneCoef& c, const OpConst& op, double mu, double2 u0, double2 sx,
                                           double2 sy, double2 zd, double2 zu) {
    const double dr = c.d + mu;
    double2 r;
    r.x = dr * u0.x - op.cx * sx.x - op.cy * sy.x - c.wd * zd.x - c.wu * zu.x;
    r.y = dr * u0.y - op.cx * sx.y - op.cy * sy.y - c.wd * zd.y - c.wu * zu.y;
    return r;
}
// planes 2 .. nz-3: theta = 1 on the plane and both z-neighbours
__device__ __forceinline__ double2 kt_int(const OpConst& op, double mu, double2 u0, double2 sx, double2 sy,
                                          double2 zs) {
    const double dr = op.dint + mu;
    double2 r;
    r.x = dr * u0.x - op.cx * sx.x - op.cy * sy.x - op.cz * zs.x;
    r.y = dr * u0.y - op.cx * sx.y - op.cy * sy.y - op.cz * zs.y;
    return r;
}

// K~ u at one node from global memory (init pass)
__device__ double2 kt_point(const OpConst& op, const double* mu, const double2* u, int i, int j, int k) {
    const size_t PS = (size_t)op.nx * op.ny;
    const size_t n = (size_t)k * PS + (size_t)j * op.nx + i;
    const double2 z = cmk(0, 0);
    const double2 w = i > 0 ? u[n - 1] : z, e = i < op.nx - 1 ? u[n + 1] : z;
    const double2 s = j > 0 ? u[n - op.nx] : z, nn = j < op.ny - 1 ? u[n + op.nx] : z;
    const double2 d = k > 0 ? u[n - PS] : z, up = k < op.nz - 1 ? u[n + PS] : z;
    const PlaneCoef c = plane_coef(op, k);
    return kt_edge(c, op, mu[n], u[n], cadd(w, e), cadd(s, nn), d, up);
}

__device__ __forceinline__ double2 cmul_re(double2 a, double s) { return make_double2(a.x * s, a.y * s); }

// ---------------------------------------------------------------- scalar recurrences
struct PairScalars {
    double2 alpha, beta;   // .x seed 0, .y seed 1 of the pair (0 for an inactive seed)
    int active;            // either seed iterates
};

// Scalars of pass k for one pair, by warp 0 of every CTA of the pair (identical, fixed-order
// reduction).  Lane l < 16 handles seed e = l / 8 and shift f = l % 8; `writer` (the first
// CTA of the pair) stores the seed states, the shift states and the fold records.
__device__ void pass_scalars(const PassArgs& a, int pair, bool writer, PairScalars* out) {
    const int lane = threadIdx.x & 31;
    const int nslots = a.tl.ntiles * a.nzch_tot;
    const double* pp = a.part[a.k & 1] + (size_t)pair * nslots * kNumPartials;
    double s[kNumPartials];
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) s[i] = 0.0;
    for (int t = lane; t < nslots; t += 32)
#pragma unroll
        for (int i = 0; i < kNumPartials; ++i) s[i] += pp[t * kNumPartials + i];
#pragma unroll
    for (int i = 0; i < kNumPartials; ++i) s[i] = warp_sum(s[i]);
    const int e = (lane >> 3) & 1, f = lane & 7;
    const int seed = 2 * pair + e;
    const int kin = (a.k + 1) & 1, kout = a.k & 1;
    const SeedState prev = a.st[kin][seed];
    SeedState cur = prev;
    const uint32_t mask = a.mask[seed];
    const bool need = lane < 16 && f < a.nshift && ((mask >> f) & 1u);
    ShiftState ss;
    ss.zp = cmk(1, 0);
    ss.zc = cmk(1, 0);
    if (need) ss = a.sh[kin][(size_t)seed * kMaxShift + f];
    // largest shifted residual factor |zeta_k|^2 over the needed shifts of this seed
    double z2 = need ? ss.zc.x * ss.zc.x + ss.zc.y * ss.zc.y : 0.0;
#pragma unroll
    for (int o = 1; o < 8; o <<= 1) z2 = fmax(z2, __shfl_xor_sync(0xffffffffu, z2, o));
    const double rho = e ? s[1] : s[0], mu = e ? s[3] : s[2], nu = e ? s[5] : s[4], sgd = e ? s[7] : s[6];
    bool act = false;
    double alpha = 0.0, beta = 0.0;
    if (!prev.done) {
        if (a.k == 0) cur.bnorm2 = rho;
        double sigma = mu;
        if (a.k > 0) {
            beta = rho / prev.rho;
            sigma = mu + 2.0 * beta * nu + beta * beta * sgd;
        }
        alpha = rho / sigma;
        if (!(z2 * rho > a.tol2 * cur.bnorm2)) {          // every needed shift converged (also b = 0)
            cur.done = 1;
            cur.iters = a.k;
        } else if (a.k >= a.max_iter) {
            cur.done = 1;
            cur.iters = a.k;
            cur.flag = DOT_ERR_NOCONV;
        } else if (!isfinite(alpha) || !isfinite(beta) || !(sigma > 0.0)) {
            cur.done = 1;
            cur.iters = a.k;
            cur.flag = DOT_ERR_BREAKDOWN;
        } else {
            act = true;
        }
    }
    if (need && writer) {
        ShiftCoef rec;
        rec.k = a.k;
        rec.active = act ? 1 : 0;
        rec.zeta = cmk(0, 0);
        rec.beta = cmk(0, 0);
        rec.alpha = cmk(0, 0);
        if (act) {
            // shifted CG (shift-invariant Krylov space): with a_{k-1} = prev.alpha (1 at k = 0),
            // zeta_{k+1} = zeta_k zeta_{k-1} a_{k-1} / (a_k b_k (zeta_{k-1} - zeta_k) + zeta_{k-1} a_{k-1} (1 + i s a_k))
            const double ap = a.k > 0 ? prev.alpha : 1.0;
            const double sg = a.sigma[f];
            const double2 zp = ss.zp, zc = ss.zc;
            const double2 den = cadd(cmul_re(csub(zp, zc), alpha * beta), cmul_re(cmul(zp, cmk(1.0, sg * alpha)), ap));
            const double2 zn = cdiv(cmul_re(cmul(zc, zp), ap), den);
            const double2 q = cdiv(zc, zp);
            rec.zeta = zc;                                   // r_sigma,k = zeta_k r_k
            rec.beta = cmul_re(cmul(q, q), beta);            // beta_sigma = (zeta_k / zeta_{k-1})^2 beta
            rec.alpha = cmul_re(cdiv(zn, zc), alpha);        // alpha_sigma = alpha zeta_{k+1} / zeta_k
            ShiftState nx;
            nx.zp = zc;
            nx.zc = zn;
            a.sh[kout][(size_t)seed * kMaxShift + f] = nx;
        }
        a.coef[((size_t)(a.k % a.hist) * (2 * a.npairs) + seed) * kMaxShift + f] = rec;
    }
    if (act) {
        cur.rho = rho;
        cur.alpha = alpha;
    } else {
        alpha = 0.0;
        beta = 0.0;
    }
    if (writer && lane < 16 && f == 0) {
        a.st[kout][seed] = cur;
        if (cur.done) a.st[kin][seed] = cur;    // a finished seed may drop out of later launches: freeze
    }
    const double a1 = __shfl_sync(0xffffffffu, alpha, 8), b1 = __shfl_sync(0xffffffffu, beta, 8);
    const int act1 = __shfl_sync(0xffffffffu, act ? 1 : 0, 8);
    if (lane == 0) {
        PairScalars sc;
        sc.alpha = cmk(alpha, a1);
        sc.beta = cmk(beta, b1);
        sc.active = (act || act1) ? 1 : 0;
        *out = sc;
    }
}

template <int I>
struct IC {
    static constexpr int v = I;
};

// Slot layout (per ring slot): r [rowsP*nx] double2 | p [rowsP*nx] double2 | mu [rowsP*nx] double
// (mu rides along in the same bulk-copy group when MUT; else it is loaded per thread).
// NX_, TY_, XS_: compile-time slot row length, tile height and x parts of the bench geometries
// (0: run time).
template <int MAXT, int NS, bool MUT, int RPT, bool ZC, int NX_, int TY_, int XS_>
__global__ void __launch_bounds__(MAXT, 1) cg_pass_kernel(const __grid_constant__ PassArgs a) {
    extern __shared__ __align__(128) unsigned char smem_raw[];
    constexpr int PD = NS - 2;                          // TMA planes in flight
    const int ntiles = a.tl.ntiles;
    const int tile = blockIdx.x % ntiles, zc = a.zc0 + blockIdx.x / ntiles;
    const int yrow = a.pair0 + (int)blockIdx.y;                    // split launches: rows [pair0, pair0 + ny)
    // programmatic dependent launch: the next pass of the stream may be scheduled now; its CTAs
    // set up their shared memory on free SMs and block at griddepcontrol.wait below until this
    // grid has completed and flushed (no-ops when launched without the attribute)
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
    // x split (wide rows): tile = (row tile ty, x part xp); the slot rows are nx = the part's
    // xw columns plus 2 halo columns on each side (local column c = global column cx0 + c)
    constexpr bool XS1 = XS_ == 1;                     // compile-time: no x split
    const int xs = XS1 ? 1 : (XS_ ? XS_ : a.tl.xs), ty = XS1 ? tile : tile / xs, xp = XS1 ? 0 : tile - ty * xs;
    const int nxg = (XS_ == 1 && NX_) ? NX_ : a.op.nx, ny = a.op.ny, nz = a.op.nz;   // global row length
    const int nx = NX_ ? NX_ : a.tl.nxl;
    const int xw = XS1 ? nxg : (nxg + xs - 1) / xs, x0 = XS1 ? 0 : xp * xw, x1 = XS1 ? nxg : min(x0 + xw, nxg);
    const int cx0 = xs > 1 ? x0 - 2 : 0;
    const int TY = TY_ ? TY_ : a.tl.TY;
    // z chunk [z0, z1) of this CTA; phase 1 runs on [a1, b1), phase 2 on [a2, b2)
    // (two / one halo planes recomputed on each side)
    const int z0 = ZC ? zc * a.zlen : 0, z1 = ZC ? min(nz, z0 + a.zlen) : nz;
    const int a1 = ZC ? max(z0 - 2, 0) : 0, b1 = ZC ? min(z1 + 2, nz) : nz;
    const int a2 = ZC ? max(z0 - 1, 0) : 0, b2 = ZC ? min(z1 + 1, nz) : nz;
    const int fend = ZC ? min(b1, z1) + 2 : nz + 2;
    const int rowsP = TY + 4, rowsR = TY + 2;
    const int PS = nxg * ny;
    const size_t N = (size_t)PS * nz;
    const int j0 = ty * TY;
    // double2 elements of one vector in a slot (x split: a multiple of 16, so that every slot and
    // each vector inside it starts 128-byte aligned for the tensor copies)
    const int slotE = xs > 1 ? (rowsP * nx + 15) / 16 * 16 : rowsP * nx;
    const int slotW = 2 * slotE + (MUT ? (slotE + 1) / 2 : 0);   // slot stride in double2
    const int rbE = rowsR * nx;

    double2* slots = reinterpret_cast<double2*>(smem_raw);          // [NS][slotW]
    double2* rbuf = slots + (size_t)NS * slotW;                     // [3][rowsR*nx]
    uint64_t* bars = reinterpret_cast<uint64_t*>(rbuf + 3 * rbE);
    // bars[0, NS): TMA ring slots; bars[NS], bars[NS + 1]: step barriers (every thread arrives after
    // its step, a warp waits for the previous step's arrivals only before reading neighbours' data)
    double* scratch = reinterpret_cast<double*>(bars + NS + 2);     // [32][kNumPartials]
    int2* s_samp = reinterpret_cast<int2*>(scratch + 32 * kNumPartials);   // [nz] sample ranges
    __shared__ PairScalars sh_sc;

    auto prologue_fill = [&]() {
        // rows outside the domain (edge tiles only) must read as zero (Dirichlet y faces):
        // the p rows of every ring slot outside [rlo, rhi) and the Rbuf rows outside
        // [rlo - 1, rhi - 1); nothing else is read before it is written
        const int rlo_ = max(0, 2 - j0), rhi_ = min(TY + 4, ny - j0 + 2);
        const int nlo = rlo_ * nx, nhi = (TY + 4 - rhi_) * nx;
        if (nlo + nhi > 0) {
            const int per = nlo + nhi;
            // (x split: every tensor copy zero-fills its box outside the domain; the prologue writes
            // nothing into the ring slots, so the first copies may be issued before the barrier)
            if (xs == 1)
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
        if (a.nP > 0)
            for (int g = threadIdx.x; g < nz; g += blockDim.x)
                s_samp[g] = XS1 ? make_int2(a.samp_off[g * ntiles + tile], a.samp_off[g * ntiles + tile + 1])
                                : make_int2(a.samp_off[g * a.tl.nty + ty], a.samp_off[g * a.tl.nty + ty + 1]);
    };
    prologue_fill();
    if (threadIdx.x == 0) {
        for (int q = 0; q < NS; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[q])), "r"(1));
        for (int q = NS; q < NS + 2; ++q)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bars[q])), "r"((int)blockDim.x));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    // everything above touches shared memory and set_params-time tables only; everything below
    // reads what the previous kernels of the stream wrote (active list, partial sums, r, p)
    asm volatile("griddepcontrol.wait;" ::: "memory");
    const int pair = a.act ? a.act[yrow] : yrow;                   // active-list compaction (tail passes)
    if (pair < 0) return;                                          // slot past the active count
    const int kin = a.k & 1, kout = kin ^ 1;      // pass 0 reads p_{-1} = 0 (zeroed buffer), beta_0 = 0
    const double2* __restrict__ Rin = a.R[kin] + (size_t)pair * N;
    const double2* __restrict__ Pin = a.Pv[kin] + (size_t)pair * N;
    double2* Hk = a.H + ((size_t)(a.k % a.hist) * a.npairs + pair) * a.nP;   // r_k at the samples

    // in-domain slot rows [rlo, rhi); grid row of slot row r is j0 - 2 + r
    const int rlo = max(0, 2 - j0), rhi = min(rowsP, ny - j0 + 2);
    const uint32_t tile_bytes = xs > 1 ? (uint32_t)(rowsP * nx * sizeof(double2))     // full box (zero fill)
                                       : (uint32_t)((rhi - rlo) * nx * sizeof(double2));
    const uint32_t mu_bytes = tile_bytes / 2;
    const uint32_t tx_bytes = 2 * tile_bytes + (MUT ? mu_bytes : 0);
    const int tile_off = (j0 - 2 + rlo) * nxg;
    const uint32_t slot0 = smem_u32(slots + rlo * nx);             // r rows of slot 0
    const uint32_t slot_stride = (uint32_t)(slotW * sizeof(double2));
    const uint32_t pvec_off = (uint32_t)(slotE * sizeof(double2));
    // mu rows land at slot + 2 slotE double2 + rlo*nx doubles (dR already includes rlo*nx double2)
    const uint32_t mu_off = (uint32_t)(2 * slotE * sizeof(double2)) - (uint32_t)(rlo * nx * 8);
    const uint32_t bar0 = smem_u32(bars);

    // one thread: bulk copies of the contiguous in-domain rows, or (x split) one tensor copy per
    // vector of the whole (TY + 4) x nxl box
    auto issue = [&](int z, int sl) {
        const uint32_t dR = slot0 + sl * slot_stride, bar = bar0 + 8 * sl;
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(tx_bytes) : "memory");
        if (xs > 1) {
            const uint32_t d0 = smem_u32(slots) + sl * slot_stride;
            const int cx = cx0, cy = j0 - 2;
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
                "[%6];" ::"r"(d0),
                "l"(reinterpret_cast<uint64_t>(&a.tmR[kin])), "r"(2 * cx), "r"(cy), "r"(z), "r"(pair), "r"(bar)
                : "memory");
            asm volatile(
                "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], "
                "[%6];" ::"r"(d0 + pvec_off),
                "l"(reinterpret_cast<uint64_t>(&a.tmP[kin])), "r"(2 * cx), "r"(cy), "r"(z), "r"(pair), "r"(bar)
                : "memory");
            if (MUT)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
                    "[%5];" ::"r"(d0 + (uint32_t)(2 * slotE * sizeof(double2))),
                    "l"(reinterpret_cast<uint64_t>(&a.tmMu)), "r"(cx), "r"(cy), "r"(z), "r"(bar)
                    : "memory");
            return;
        }
        const size_t g = (size_t)z * PS + tile_off;
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dR),
            "l"(Rin + g), "r"(tile_bytes), "r"(bar)
            : "memory");
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
    // First planes: the copies land in slot rows no thread writes in the prologue (unsplit rows: the
    // in-domain rows; x split: whole boxes, which the prologue leaves alone), so thread 0 issues them
    // before the scalars and the copy latency overlaps pass_scalars and the barrier.
    int npre = 0;
    if (threadIdx.x == 0)
        for (int z = a1; z < a1 + PD && z < b1; ++z, ++npre) issue(z, z - a1);
    if (threadIdx.x < 32) pass_scalars(a, pair, blockIdx.x == 0, &sh_sc);
    __syncthreads();
    if (!sh_sc.active) {
        // a finished pair still in the launch: the copies in flight must land before the CTA exits
        if (threadIdx.x == 0)
            for (int q = 0; q < npre; ++q)
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "WAITX_%=:\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                    "@!p bra WAITX_%=;\n\t}" ::"r"(bar0 + 8 * q),
                    "r"(0)
                    : "memory");
        return;
    }

    // ---- per-thread geometry: rows r0 .. r0 + RPT - 1 of column x
    const int t = threadIdx.x;
    const int m = t / nx, x = t - m * nx;
    const int r0 = RPT * m;
    const int xg = cx0 + x;                            // global column
    const bool inx = XS1 || (xg >= 0 && xg < nxg), ownx = XS1 || (xg >= x0 && xg < x1);
    const bool ph2x = XS1 || (xg >= x0 - 1 && xg <= x1);
    bool indom[RPT], own[RPT], ph2[RPT];
    bool any_in = false, any2 = false, any_own = false;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        const int r = r0 + j;
        indom[j] = r < rowsP && r >= rlo && r < rhi && inx;
        own[j] = indom[j] && r >= 2 && r < TY + 2 && ownx;
        ph2[j] = XS1 ? (own[j] || (indom[j] && (r == 1 || r == TY + 2))) : (indom[j] && r >= 1 && r <= TY + 2 && ph2x);
        any_in |= indom[j];
        any2 |= ph2[j];
        any_own |= own[j];
    }
    bool all_in = true, all2 = true;
#pragma unroll
    for (int j = 0; j < RPT; ++j) {
        all_in &= indom[j];
        all2 &= ph2[j];
    }
    const int o = r0 * nx + x;                         // slot element of row 0
    const int o3 = o - nx;                             // Rbuf element of row 0
    const int go = (j0 - 2 + r0) * nxg + xg;           // plane offset of row 0 (may be outside; unused then)
    const bool hasW = xg > 0, hasE = xg < nxg - 1;
    // running per-thread global pointers (advance one plane per step)
    double2* pP = a.Pv[kout] + (size_t)pair * N + go + (ptrdiff_t)a1 * PS;        // p_k at plane f
    double2* pR = a.R[kout] + (size_t)pair * N + go + (ptrdiff_t)(a1 - 2) * PS;   // r_{k+1} at plane f - 2
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
    int sidx = 0;                      // step counter (step barrier = bars[NS + (sidx & 1)])
    const uint32_t sbar0 = bar0 + 8 * NS;

    auto step = [&](int f, auto IDX) {
        constexpr int i0 = decltype(IDX)::v;           // f % 3
        constexpr int i1 = (i0 + 2) % 3;               // (f - 1) % 3
        constexpr int i2 = (i0 + 1) % 3;               // (f - 2) % 3
        const bool ownf = !ZC || (f >= z0 && f < z1);
        if (!MUT && f < b1)
#pragma unroll
            for (int j = 0; j < RPT; ++j)
                if (ph2[j]) MU[j][i0] = pMu[(size_t)f * PS + j * nxg];
        // ---- phase 1: plane f
        // (zeros are assigned only on the paths that need them: rows outside the domain, and
        // the tail steps past the last plane -- no per-step register clears)
        double2 pf[RPT];
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
                        if (!A && !indom[j]) {
                            pf[j] = z2;
                            continue;
                        }
                        const double2 rf = sr[j * nx];
                        const double2 pv = sr[slotE + j * nx];
                        pf[j] = cmk(fma(beta.x, pv.x, rf.x), fma(beta.y, pv.y, rf.y));
                        sr[slotE + j * nx] = pf[j];
                        if (own[j] && ownf) pP[j * nxg] = pf[j];
                    }
                };
                if (all_in) p1(IC<1>());
                else p1(IC<0>());
            } else {
#pragma unroll
                for (int j = 0; j < RPT; ++j) pf[j] = z2;
            }
        } else {
#pragma unroll
            for (int j = 0; j < RPT; ++j) pf[j] = z2;
        }
        // ---- every thread's step f-1 (smem p of plane f-1, Rbuf of plane f-2, reads of the ring slot
        // of plane f-2) must be complete before phase 2 reads neighbours and before that slot is
        // refilled; phase 1 above only touched this thread's own rows of the plane-f slot
        if (sidx > 0) {
            const int ps = sidx - 1;
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "WAITS_%=:\n\t"
                "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
                "@!p bra WAITS_%=;\n\t}" ::"r"(sbar0 + 8 * (ps & 1)),
                "r"((ps >> 1) & 1)
                : "memory");
        }
        if (threadIdx.x == 0 && f + PD < b1) issue(f + PD, sl_iss);
        // ---- phase 2: plane g = f - 1
        double2 rng[RPT];
        double mug[RPT];           // read (phase 3 via mu_carry) only for rows that assign it
        const int g = f - 1;
        if (g >= a2 && g < b2) {
            const bool owng = !ZC || (g >= z0 && g < z1);
            const double2* sr = slots + sl_prev * slotW;
            const double2* sp = sr + slotE;
            if (any2) {
                const bool interior = g > 1 && g < nz - 2;
                const PlaneCoef ce = interior ? PlaneCoef{} : edge_coef(a, g);
                const double2 alpha = sh_sc.alpha;
                auto p2 = [&](auto ALL) {
                    constexpr bool A = decltype(ALL)::v != 0;
#pragma unroll
                    for (int j = 0; j < RPT; ++j) {
                        if (!A && !ph2[j]) {
                            rng[j] = z2;
                            continue;
                        }
                        const int oj = o + j * nx;
                        const double2 vw = sp[oj - 1], ve = sp[oj + 1];   // unconditional: selects, not branches
                        const double2 xw = hasW ? vw : z2;
                        const double2 xe = hasE ? ve : z2;
                        const double2 ys = j > 0 ? Pq[j > 0 ? j - 1 : 0][i1] : sp[oj - nx];
                        const double2 yn = j < RPT - 1 ? Pq[j < RPT - 1 ? j + 1 : 0][i1] : sp[oj + nx];
                        mug[j] = MUT ? reinterpret_cast<const double*>(sr + 2 * slotE)[oj] : MU[j][i1];
                        const double2 pc = Pq[j][i1];
                        double2 qv;
                        if (interior)
                            qv = kt_int(a.op, mug[j], pc, cadd(xw, xe), cadd(ys, yn), cadd(Pq[j][i2], pf[j]));
                        else
                            qv = kt_edge(ce, a.op, mug[j], pc, cadd(xw, xe), cadd(ys, yn), Pq[j][i2], pf[j]);
                        const double2 rk = sr[oj];
                        rng[j] = cmk(fma(-alpha.x, qv.x, rk.x), fma(-alpha.y, qv.y, rk.y));
                        rbuf[i1 * rbE + o3 + j * nx] = rng[j];
                        if (own[j] && owng) {
                            acc[4] = fma(rng[j].x, qv.x, acc[4]);
                            acc[5] = fma(rng[j].y, qv.y, acc[5]);
                            acc[6] = fma(pc.x, qv.x, acc[6]);
                            acc[7] = fma(pc.y, qv.y, acc[7]);
                        }
                    }
                };
                if (all2) p2(IC<1>());
                else p2(IC<0>());
            } else {
#pragma unroll
                for (int j = 0; j < RPT; ++j) rng[j] = z2;
            }
            if (a.nP > 0 && owng) {        // r_k at the samples of plane g (history for the fold)
                const int2 sr2 = s_samp[g];
                for (int si = sr2.x + threadIdx.x; si < sr2.y; si += blockDim.x) {
                    const int rem = a.samp_nodes[si] - g * PS;
                    if (xs == 1) {
                        Hk[si] = sr[rem - (j0 - 2) * nx];
                    } else {
                        const int row = rem / nxg, col = rem - row * nxg;
                        if (col >= x0 && col < x1) Hk[si] = sr[(row - (j0 - 2)) * nx + (col - cx0)];
                    }
                }
            }
        } else {
#pragma unroll
            for (int j = 0; j < RPT; ++j) rng[j] = z2;
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) Pq[j][i0] = pf[j];
        // this step's shared-memory writes are done (phase 3 writes only registers and HBM): arrive.
        // The next step's waits then also cover this thread's phase-3 reads of Rbuf plane f - 2,
        // which is rewritten two steps later only.
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sbar0 + 8 * (sidx & 1)) : "memory");
        // ---- phase 3: plane tt = f - 2
        const int tt = f - 2;
        if (any_own && tt >= z0 && tt < z1) {
            const double2* rc = rbuf + i2 * rbE + o3;
            const bool interior = tt > 1 && tt < nz - 2;
            const PlaneCoef ce = interior ? PlaneCoef{} : edge_coef(a, tt);
#pragma unroll
            for (int j = 0; j < RPT; ++j) {
                if (!own[j]) continue;
                const double2 vw = rc[j * nx - 1], ve = rc[j * nx + 1];
                const double2 xw = hasW ? vw : z2;
                const double2 xe = hasE ? ve : z2;
                // y-neighbours: own-strip rows from registers (r_{k+1} of plane tt is RN[.][i2])
                const double2 ys = j > 0 ? RN[j > 0 ? j - 1 : 0][i2] : rc[(j - 1) * nx];
                const double2 yn = j < RPT - 1 ? RN[j < RPT - 1 ? j + 1 : 0][i2] : rc[(j + 1) * nx];
                const double2 r0v = RN[j][i2];
                const double mut = MUT ? mu_carry[j] : MU[j][i2];
                double2 ar;
                if (interior)
                    ar = kt_int(a.op, mut, r0v, cadd(xw, xe), cadd(ys, yn), cadd(RN[j][i0], rng[j]));
                else
                    ar = kt_edge(ce, a.op, mut, r0v, cadd(xw, xe), cadd(ys, yn), RN[j][i0], rng[j]);
                acc[0] = fma(r0v.x, r0v.x, acc[0]);
                acc[1] = fma(r0v.y, r0v.y, acc[1]);
                acc[2] = fma(r0v.x, ar.x, acc[2]);
                acc[3] = fma(r0v.y, ar.y, acc[3]);
                pR[j * nxg] = r0v;
            }
        }
#pragma unroll
        for (int j = 0; j < RPT; ++j) {
            RN[j][i1] = rng[j];
            mu_carry[j] = mug[j];
        }
        pP += PS;
        pR += PS;
        sl_prev = sl;
        if (++sl == NS) {
            sl = 0;
            par ^= 1u;
        }
        if (++sl_iss == NS) sl_iss = 0;
        ++sidx;
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
    for (int i = 0; i < kNumPartials; ++i) acc[i] = warp_sum(acc[i]);
    if (lane == 0)
#pragma unroll
        for (int i = 0; i < kNumPartials; ++i) scratch[warp * kNumPartials + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < kNumPartials) {
        double sum = 0;
        for (int w = 0; w < nw; ++w) sum += scratch[w * kNumPartials + threadIdx.x];
        a.part[kout][((size_t)pair * ntiles * a.nzch_tot + (size_t)zc * ntiles + tile) * kNumPartials + threadIdx.x] =
            sum;
    }
}

// partials[0] of every pair: rho_0 = b~^T b~, mu_0 = b~^T K~ b~ (tile-owned rows, all planes);
// seed / shift states of "pass -1": not done, zeta_{-1} = zeta_0 = 1
__global__ void __launch_bounds__(256) cg_init_kernel(const PassArgs a, int zc_own) {
    __shared__ double scratch[8 * kNumPartials];
    const int tile = blockIdx.x, pair = blockIdx.y;
    const int nx = a.op.nx, ny = a.op.ny, nz = a.op.nz;
    const size_t N = (size_t)nx * ny * nz;
    const int j0 = tile * a.tl.TY, ty_own = min(a.tl.TY, ny - j0);
    const double2* b = a.R[0] + (size_t)pair * N;
    double acc[kNumPartials];
    for (int i = 0; i < kNumPartials; ++i) acc[i] = 0;
    const int per_plane = ty_own * nx;
    for (int idx = threadIdx.x; idx < per_plane * nz; idx += blockDim.x) {
        const int k = idx / per_plane, rem = idx - k * per_plane;
        const int j = j0 + rem / nx, i = rem % nx;
        const double2 r0 = b[((size_t)k * ny + j) * nx + i];
        if (r0.x == 0.0 && r0.y == 0.0) continue;
        const double2 ar = kt_point(a.op, a.mu, b, i, j, k);
        acc[0] = fma(r0.x, r0.x, acc[0]);
        acc[1] = fma(r0.y, r0.y, acc[1]);
        acc[2] = fma(r0.x, ar.x, acc[2]);
        acc[3] = fma(r0.y, ar.y, acc[3]);
    }
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int i = 0; i < kNumPartials; ++i) acc[i] = warp_sum(acc[i]);
    if (lane == 0)
        for (int i = 0; i < kNumPartials; ++i) scratch[warp * kNumPartials + i] = acc[i];
    __syncthreads();
    if (threadIdx.x < kNumPartials) {
        double s = 0;
        for (int w = 0; w < nw; ++w) s += scratch[w * kNumPartials + threadIdx.x];   // fixed order
        // the slot (zc_own, tile) carries the sums; every other z-chunk slot of the pair is zero
        double* out = a.part[0] + (size_t)pair * a.tl.ntiles * a.nzch_tot * kNumPartials;
        for (int zc = 0; zc < a.nzch_tot; ++zc)
            out[((size_t)zc * a.tl.ntiles + tile) * kNumPartials + threadIdx.x] = zc == zc_own ? s : 0.0;
    }
    if (tile == 0 && threadIdx.x < 2) {
        const int seed = 2 * pair + threadIdx.x;
        SeedState s0{};
        a.st[1][seed] = s0;     // pass 0 reads st[1]: not done
        for (int f = 0; f < kMaxShift; ++f) {
            ShiftState z;
            z.zp = cmk(1, 0);
            z.zc = cmk(1, 0);
            a.sh[1][(size_t)seed * kMaxShift + f] = z;
        }
    }
}

// Fold of passes [k0, k1) into the shifted directions and solutions on the samples
// [s0, s1): thread (pair, sample) runs both seeds' recurrences in pass order.
template <int NSL>
__global__ void __launch_bounds__(128) cg_fold_kernel(FoldArgs f) {
    // the fold records of this pair's two seeds for passes [k0, k1), valid flags folded in
    __shared__ double2 sc[2][kHist][NSL][3];      // zeta, beta_sigma, alpha_sigma
    __shared__ int sv[2][kHist][NSL];
    const int pair = blockIdx.y;
    const int nk = f.k1 - f.k0, nseeds = 2 * f.npairs;
    for (int i = threadIdx.x; i < 2 * nk * NSL; i += blockDim.x) {
        const int e = i / (nk * NSL), rem = i - e * nk * NSL, kk = rem / NSL, sl = rem - kk * NSL;
        const int seed = 2 * pair + e, k = f.k0 + kk;
        uint32_t m = f.mask[seed];
        int q = -1;
        for (int c = 0; m; ++c) {                  // sl-th needed shift of the seed
            const int b = __ffs(m) - 1;
            m &= m - 1;
            if (c == sl) {
                q = b;
                break;
            }
        }
        int valid = 0;
        if (q >= 0 && q < f.nshift) {
            const ShiftCoef c = f.coef[((size_t)(k % f.hist) * nseeds + seed) * kMaxShift + q];
            valid = (c.k == k && c.active) ? 1 : 0;
            sc[e][kk][sl][0] = c.zeta;
            sc[e][kk][sl][1] = c.beta;
            sc[e][kk][sl][2] = c.alpha;
        }
        sv[e][kk][sl] = valid;
    }
    __syncthreads();
    const int s = f.s0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= f.s1) return;
    const uint32_t m0 = f.mask[2 * pair], m1 = f.mask[2 * pair + 1];
    const int n0 = min(__popc(m0), NSL), n1 = min(__popc(m1), NSL);
    double2 Pv[2][NSL], Xv[2][NSL];
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl) {
            Pv[e][sl] = cmk(0, 0);
            Xv[e][sl] = cmk(0, 0);
            if (sl < (e ? n1 : n0)) {
                const size_t ix = ((size_t)(2 * pair + e) * f.nsl + sl) * f.nP + s;
                Pv[e][sl] = f.Ps[ix];
                Xv[e][sl] = f.Xs[ix];
            }
        }
#pragma unroll 1
    for (int kk = 0; kk < nk; ++kk) {
        const int k = f.k0 + kk;
        const double2 hv = f.H[((size_t)(k % f.hist) * f.npairs + pair) * f.nP + s];
#pragma unroll
        for (int e = 0; e < 2; ++e) {
            const double r = e ? hv.y : hv.x;
#pragma unroll
            for (int sl = 0; sl < NSL; ++sl) {
                if (!sv[e][kk][sl]) continue;
                Pv[e][sl] = cfma(sc[e][kk][sl][1], Pv[e][sl], cmul_re(sc[e][kk][sl][0], r));
                Xv[e][sl] = cfma(sc[e][kk][sl][2], Pv[e][sl], Xv[e][sl]);
            }
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e)
#pragma unroll
        for (int sl = 0; sl < NSL; ++sl)
            if (sl < (e ? n1 : n0)) {
                const size_t ix = ((size_t)(2 * pair + e) * f.nsl + sl) * f.nP + s;
                f.Ps[ix] = Pv[e][sl];
                f.Xs[ix] = Xv[e][sl];
            }
}

// XP[obase + q*ostride][s] += mul * theta^-1/2 * Xs[seed][q][s] over the seeds' needed shifts
__global__ void __launch_bounds__(128) cg_finalize_kernel(FoldArgs f, OpConst op, double2* XP, int nP_out,
                                                         const int32_t* omap, const int32_t* samp_nodes) {
    const int pair = blockIdx.y;
    const int s = f.s0 + blockIdx.x * blockDim.x + threadIdx.x;
    if (s >= f.s1) return;
    const int PS = op.nx * op.ny;
    const double us = unscale_of(samp_nodes[s] / PS, op.nz);
    for (int e = 0; e < 2; ++e) {
        const int seed = 2 * pair + e;
        const uint32_t mask = f.mask[seed];
        const int obase = omap[3 * seed], ostride = omap[3 * seed + 1], imag = omap[3 * seed + 2];
        if (!mask || obase < 0) continue;
        for (int q = 0; q < f.nshift; ++q) {
            if (!((mask >> q) & 1u)) continue;
            const double2 v = cmul_re(f.Xs[((size_t)seed * f.nsl + __popc(mask & ((1u << q) - 1u))) * f.nP + s], us);
            double2* dst = XP + (size_t)(obase + q * ostride) * nP_out + s;
            const double2 cur = *dst;
            *dst = imag ? cmk(cur.x - v.y, cur.y + v.x) : cadd(cur, v);
        }
    }
}

__global__ void apply_kernel(OpConst op, const double* mu, const double* shift, const double2* u, double2* Au,
                             int nb) {
    // A(omega, p) u in the unscaled variables (Eq. (2.1), R1-R3):
    //   theta_k [cx (2u - uW - uE) + cy (2u - uS - uN) + (mu + i shift) u] + cz (nzn u - uD - uU) + robin_k u
    const size_t N = (size_t)op.nx * op.ny * op.nz;
    const size_t PS = (size_t)op.nx * op.ny;
    const int rhs = blockIdx.y;
    const double2* v = u + (size_t)rhs * N;
    for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += (size_t)gridDim.x * blockDim.x) {
        const int i = n % op.nx, j = (n / op.nx) % op.ny, k = n / PS;
        const double2 z = cmk(0, 0);
        const double2 w = i > 0 ? v[n - 1] : z, e = i < op.nx - 1 ? v[n + 1] : z;
        const double2 s = j > 0 ? v[n - op.nx] : z, nn = j < op.ny - 1 ? v[n + op.nx] : z;
        const double2 d = k > 0 ? v[n - PS] : z, up = k < op.nz - 1 ? v[n + PS] : z;
        const double th = (k == 0 || k == op.nz - 1) ? 0.5 : 1.0;
        const double nzn = (k > 0 ? 1.0 : 0.0) + (k < op.nz - 1 ? 1.0 : 0.0);
        const double rob = (k == 0 || k == op.nz - 1) ? op.robin : 0.0;
        const double2 u0 = v[n];
        const double dre = th * (2.0 * op.cx + 2.0 * op.cy + mu[n]) + op.cz * nzn + rob;
        const double dim = th * shift[rhs];
        double2 r;
        r.x = dre * u0.x - dim * u0.y - th * (op.cx * (w.x + e.x) + op.cy * (s.x + nn.x)) - op.cz * (d.x + up.x);
        r.y = dre * u0.y + dim * u0.x - th * (op.cx * (w.y + e.y) + op.cy * (s.y + nn.y)) - op.cz * (d.y + up.y);
        Au[(size_t)rhs * N + n] = r;
    }
}

__global__ void count_active_kernel(const SeedState* st, int npairs, int* out, int32_t* act) {
    // one block: ordered compaction of the pairs with a seed still iterating
    __shared__ int wsum[32];
    __shared__ int base;
    if (threadIdx.x == 0) base = 0;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int c0 = 0; c0 < npairs; c0 += blockDim.x) {
        const int r = c0 + threadIdx.x;
        const int a = (r < npairs && !(st[2 * r].done && st[2 * r + 1].done)) ? 1 : 0;
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
    if (act)   // entries past the count: no pair (a pass launched with an older, larger count skips them)
        for (int y = base + threadIdx.x; y < npairs; y += blockDim.x) act[y] = -1;
    if (threadIdx.x == 0) *out = base;
}

// R0[pair][node[a]].(x|y) = coeff[a*ncols + c] * scale[a] * theta^-1/2 for a run of seeds
__global__ void scatter_seed_kernel(double2* R0, size_t N, const int32_t* nodes, int nnodes, const double* coeff,
                                    int ncols, const double* scale, int col0, int seed0, int PS, int nz) {
    const int ls = seed0 + blockIdx.x;         // chunk-local seed
    const int c = col0 + blockIdx.x;
    double* dst = reinterpret_cast<double*>(R0 + (size_t)(ls >> 1) * N) + (ls & 1);
    for (int a = threadIdx.x; a < nnodes; a += blockDim.x) {
        const double w = coeff ? coeff[(size_t)a * ncols + c] : (a == c ? 1.0 : 0.0);
        if (w != 0.0) {
            const int n = nodes[a];
            dst[2 * (size_t)n] = w * scale[a] * unscale_of(n / PS, nz);
        }
    }
}

// dense complex right-hand side r -> seeds (Re, Im) of pair r, scaled by theta^-1/2
__global__ void split_dense_kernel(double2* R0, const double2* b, size_t N, int PS, int nz) {
    const int r = blockIdx.y;
    for (size_t n = blockIdx.x * (size_t)blockDim.x + threadIdx.x; n < N; n += (size_t)gridDim.x * blockDim.x) {
        const double us = unscale_of((int)(n / PS), nz);
        const double2 v = b[(size_t)r * N + n];
        R0[(size_t)r * N + n] = cmk(v.x * us, v.y * us);
    }
}

// z-slab halo: buf[v][pair][j][PS] <-> planes z0 + j of vector v (0: r, 1: p) of every pair
__global__ void pack_planes_kernel(const double2* A, const double2* B, size_t N, int PS, int z0, int n,
                                   double2* buf, int unpack, double2* Aw, double2* Bw) {
    const int pair = blockIdx.y, v = blockIdx.z;
    const size_t per = (size_t)n * PS;
    double2* b = buf + ((size_t)v * gridDim.y + pair) * per;
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < per; i += (size_t)gridDim.x * blockDim.x) {
        const size_t g = (size_t)pair * N + (size_t)z0 * PS + i;
        if (unpack) (v ? Bw : Aw)[g] = b[i];
        else b[i] = (v ? B : A)[g];
    }
}

}  // namespace

size_t pass_smem(int nx, int TY, int NS, int nz, bool mut, int xs = 1) {
    const size_t slotE = xs > 1 ? ((size_t)(TY + 4) * nx + 15) / 16 * 16 : (size_t)(TY + 4) * nx;
    const size_t e = (size_t)NS * (2 * slotE + (mut ? (slotE + 1) / 2 : 0)) + 3 * (size_t)(TY + 2) * nx;
    return e * sizeof(double2) + (NS + 2) * 8 + 32 * kNumPartials * 8 + 8 * (size_t)nz + 128;
}

// Pass tiling: a thread owns `rows` slot rows of one column of the TY + 4 slot rows.
//   2 rows per thread, <= 512 threads (default);  1 row per thread, <= 512 threads (fallback)
// Wide rows (nx >= 96) may split each row tile into xs = 2 x parts of ceil(nx / 2) columns plus
// 2 halo columns per side: the 512-thread / 227 KB limits then allow a taller tile, and the
// redundant halo work per owned node, (TY + 4) / TY * nxl / (nx / xs), drops (96^3: TY 6 -> 14,
// 1.67 -> 1.39).  Among the allowed x splits the tiling with the smaller halo factor wins.
// DOT_CG_TY forces the tile height, DOT_CG_ROWS the rows per thread, DOT_CG_PREFETCH the TMA
// depth (1..3), DOT_CG_XS the x parts -- test knobs.
CgTiling cg_tiling(int nx, int ny, int nz, int prefetch, int want_ty, int want_rows, bool no_mu, int want_xs) {
    const int NS = std::max(1, std::min(prefetch, 3)) + 2;
    const size_t sm_cta = 227 * 1024;
    struct Opt { int rows, maxt; };
    const Opt opts[2] = {{2, 512}, {1, 512}};
    CgTiling best;
    bool found = false;
    double best_cost = 0;
    for (int xs = 1; xs <= 2; ++xs) {
        if (want_xs > 0 && xs != want_xs) continue;
        // x parts of even width (16-byte tensor rows); by default only for 96 <= nx < 128, where it
        // measured faster (opt96 10-pair batches 0.47 -> 0.53 of the HBM peak); at nx = 128 the
        // unsplit TY = 4 tile measured faster (0.589 vs 0.561), DESIGN.md "x split"
        if (xs == 2 && nx % 4 != 0) continue;
        if (xs == 2 && want_xs != 2 && (nx < 96 || nx >= 128)) continue;
        const int nxl = xs == 1 ? nx : (nx + 1) / 2 + 4;
        const bool mut = (nxl % 2 == 0) && (nx % 2 == 0) && !no_mu;    // mu in the slots needs 16-byte rows
        CgTiling bx;
        bool fx = false;
        for (const Opt& o : opts) {
            if (want_rows > 0 && o.rows != want_rows) continue;
            int ty = 0;
            for (int c = 1; c <= ny; ++c) {
                const int thr = ((c + 4 + o.rows - 1) / o.rows * nxl + 31) / 32 * 32;
                if (thr > o.maxt || pass_smem(nxl, c, NS, nz, mut, xs) > sm_cta) break;
                ty = c;
                if (want_ty > 0 && c == want_ty) break;
            }
            if (want_ty > 0 && ty != want_ty) continue;
            if (ty <= 0) continue;
            const int nty = (ny + ty - 1) / ty;
            CgTiling t;
            t.rows = o.rows;
            t.TY = (ny + nty - 1) / nty;      // balanced tiles
            t.nty = (ny + t.TY - 1) / t.TY;
            t.xs = xs;
            t.nxl = nxl;
            t.ntiles = t.nty * xs;
            t.nslots = NS;
            t.threads = ((t.TY + 4 + o.rows - 1) / o.rows * nxl + 31) / 32 * 32;
            t.smem = pass_smem(nxl, t.TY, NS, nz, mut, xs);
            t.mut = mut;
            if (!fx || (bx.TY < 4 && t.TY > bx.TY)) {
                bx = t;
                fx = true;
            }
            if (bx.TY >= 4 || want_ty > 0) break;
        }
        if (!fx) continue;
        const double cost = (double)(bx.TY + 4) / bx.TY * (double)bx.nxl / ((double)nx / xs);
        if (!found || cost < best_cost - 1e-9) {
            best = bx;
            best_cost = cost;
            found = true;
        }
    }
    if (!found) throw Error(DOT_ERR_ARG, "no pass tiling fits this grid (nx too large or forced tile height)");
    return best;
}

template <int MAXT, int NS, int RPT>
static void launch_pass_ns(const PassArgs& a, int nb, cudaStream_t s) {
    // mu rides in the bulk-copy group when every copy is 16-byte sized and aligned
    const bool mut = a.tl.mut;
    const bool zc = a.nzch > 1 || a.nzch_tot > 1;
    using KF = void (*)(const PassArgs);
    KF k = mut ? (zc ? cg_pass_kernel<MAXT, NS, true, RPT, true, 0, 0, 0> : cg_pass_kernel<MAXT, NS, true, RPT, false, 0, 0, 0>)
               : (zc ? cg_pass_kernel<MAXT, NS, false, RPT, true, 0, 0, 0>
                     : cg_pass_kernel<MAXT, NS, false, RPT, false, 0, 0, 0>);
    // compile-time geometries of the BASELINE grids (default ring depth, 2 rows per thread)
    if constexpr (NS == 4 && RPT == 2) if (mut && !std::getenv("DOT_CG_GENERIC")) {
#define DOT_GEOM(GX, GT, GS)                                                                     \
    if (a.tl.nxl == GX && a.tl.TY == GT && a.tl.xs == GS)                                        \
        k = zc ? cg_pass_kernel<MAXT, NS, true, RPT, true, GX, GT, GS>                           \
               : cg_pass_kernel<MAXT, NS, true, RPT, false, GX, GT, GS>;
        DOT_GEOM(32, 16, 1)
        DOT_GEOM(64, 11, 1)
        DOT_GEOM(52, 14, 2)     // 96^3, two x parts
        DOT_GEOM(128, 4, 1)
#undef DOT_GEOM
    }
    ensure_smem(k, a.tl.smem);
    dim3 grid(a.tl.ntiles * a.nzch, nb);
    // programmatic dependent launch: a pass that follows a pass
    // in the stream is scheduled while its predecessor drains (tl.pdl; DOT_CG_PDL=0 at dot_create launches plainly)
    cudaLaunchConfig_t lc = {};
    lc.gridDim = grid;
    lc.blockDim = dim3(a.tl.threads);
    lc.dynamicSmemBytes = a.tl.smem;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    lc.attrs = at;
    lc.numAttrs = a.tl.pdl ? 1 : 0;
    DOT_CUDA_TRY(cudaLaunchKernelEx(&lc, k, a));
    DOT_CUDA_TRY(cudaGetLastError());
}

template <int MAXT, int RPT>
static void launch_pass_r(const PassArgs& a, int nb, cudaStream_t s) {
    switch (a.tl.nslots) {
        case 3: launch_pass_ns<MAXT, 3, RPT>(a, nb, s); break;
        case 4: launch_pass_ns<MAXT, 4, RPT>(a, nb, s); break;
        case 5: launch_pass_ns<MAXT, 5, RPT>(a, nb, s); break;
        default: throw Error(DOT_ERR_ARG, "pass supports 3..5 ring slots");
    }
}

static PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = [] {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        DOT_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        if (!p || q != cudaDriverEntryPointSuccess) throw Error(DOT_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }();
    return fn;
}

void set_pass_tmaps(PassArgs& a) {
    if (a.tl.xs <= 1) return;
    auto enc = tmap_encoder();
    const cuuint64_t nx = (cuuint64_t)a.op.nx, ny = (cuuint64_t)a.op.ny, nz = (cuuint64_t)a.op.nz;
    const cuuint32_t rows = (cuuint32_t)(a.tl.TY + 4), cols = (cuuint32_t)a.tl.nxl;
    auto check = [](CUresult r) {
        if (r != CUDA_SUCCESS) throw Error(DOT_ERR_CUDA, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")");
    };
    const cuuint64_t dim4[4] = {2 * nx, ny, nz, (cuuint64_t)std::max(a.npairs, 1)};
    const cuuint64_t str4[3] = {2 * nx * 8, 2 * nx * ny * 8, 2 * nx * ny * nz * 8};
    const cuuint32_t box4[4] = {2 * cols, rows, 1, 1}, es4[4] = {1, 1, 1, 1};
    for (int i = 0; i < 2; ++i) {
        check(enc(&a.tmR[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a.R[i], dim4, str4, box4, es4,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        check(enc(&a.tmP[i], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, a.Pv[i], dim4, str4, box4, es4,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
    }
    if (!a.tl.mut) return;                       // mu is then loaded per thread
    const cuuint64_t dim3_[3] = {nx, ny, nz};
    const cuuint64_t str3[2] = {nx * 8, nx * ny * 8};
    const cuuint32_t box3[3] = {cols, rows, 1}, es3[3] = {1, 1, 1};
    check(enc(&a.tmMu, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<double*>(a.mu), dim3_, str3, box3, es3,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
}

void set_edge_coefs(PassArgs& a) {
    const int kk[4] = {0, std::min(1, a.op.nz - 1), std::max(a.op.nz - 2, 0), a.op.nz - 1};
    for (int i = 0; i < 4; ++i) {
        const PlaneCoef c = plane_coef(a.op, kk[i]);
        a.ec[i][0] = c.d;
        a.ec[i][1] = c.wd;
        a.ec[i][2] = c.wu;
    }
}

void launch_cg_pass(const PassArgs& a, int nb, cudaStream_t s) {
    if (a.tl.rows == 2) launch_pass_r<512, 2>(a, nb, s);
    else launch_pass_r<512, 1>(a, nb, s);
}

void launch_cg_init(const PassArgs& a, int nb, cudaStream_t s, int zc_own) {
    dim3 grid(a.tl.ntiles, nb);
    cg_init_kernel<<<grid, 256, 0, s>>>(a, zc_own);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_cg_fold(const FoldArgs& f, cudaStream_t s) {
    if (f.k1 <= f.k0 || f.s1 <= f.s0 || f.npairs <= 0) return;
    if (f.k1 - f.k0 > kHist || f.hist > 2 * kHist) throw Error(DOT_ERR_ARG, "fold span exceeds the history ring");
    dim3 grid((f.s1 - f.s0 + 127) / 128, f.npairs);
    switch (f.nsl) {
        case 1: cg_fold_kernel<1><<<grid, 128, 0, s>>>(f); break;
        case 2: cg_fold_kernel<2><<<grid, 128, 0, s>>>(f); break;
        case 3: cg_fold_kernel<3><<<grid, 128, 0, s>>>(f); break;
        case 4: cg_fold_kernel<4><<<grid, 128, 0, s>>>(f); break;
        case 5: cg_fold_kernel<5><<<grid, 128, 0, s>>>(f); break;
        case 6: cg_fold_kernel<6><<<grid, 128, 0, s>>>(f); break;
        case 7: cg_fold_kernel<7><<<grid, 128, 0, s>>>(f); break;
        case 8: cg_fold_kernel<8><<<grid, 128, 0, s>>>(f); break;
        default: throw Error(DOT_ERR_ARG, "fold: 1..8 shifts per seed");
    }
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_cg_finalize(const FoldArgs& f, const OpConst& op, double2* XP, int nP_out, const int32_t* omap,
                        const int32_t* samp_nodes, cudaStream_t s) {
    if (f.s1 <= f.s0 || f.npairs <= 0) return;
    dim3 grid((f.s1 - f.s0 + 127) / 128, f.npairs);
    cg_finalize_kernel<<<grid, 128, 0, s>>>(f, op, XP, nP_out, omap, samp_nodes);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_count_active(const SeedState* st, int npairs, int* d_count, cudaStream_t s, int32_t* act) {
    count_active_kernel<<<1, 256, 0, s>>>(st, npairs, d_count, act);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_apply(const OpConst& op, const double* mu, const double* shift, const double2* u, double2* Au, int nb,
                  cudaStream_t s) {
    const size_t N = (size_t)op.nx * op.ny * op.nz;
    dim3 grid((unsigned)std::min<size_t>((N + 255) / 256, 4096), nb);
    apply_kernel<<<grid, 256, 0, s>>>(op, mu, shift, u, Au, nb);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_scatter_seeds(double2* R0, size_t N, const int32_t* nodes, int nnodes, const double* coeff, int ncols,
                          const double* scale, int col0, int seed0, int nseeds, const OpConst& op, cudaStream_t s) {
    if (nseeds <= 0) return;
    scatter_seed_kernel<<<nseeds, 128, 0, s>>>(R0, N, nodes, nnodes, coeff, ncols, scale, col0, seed0, op.nx * op.ny,
                                               op.nz);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_split_dense(double2* R0, const double2* b, size_t N, int nr, const OpConst& op, cudaStream_t s) {
    if (nr <= 0) return;
    dim3 grid((unsigned)std::min<size_t>((N + 255) / 256, 2048), nr);
    split_dense_kernel<<<grid, 256, 0, s>>>(R0, b, N, op.nx * op.ny, op.nz);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_pack_planes(const double2* R, const double2* Pv, int npairs, size_t N, int PS, int z0, int n,
                        double2* buf, cudaStream_t s) {
    if (n <= 0 || npairs <= 0) return;
    dim3 grid((unsigned)std::min<size_t>(((size_t)n * PS + 255) / 256, 512), npairs, 2);
    pack_planes_kernel<<<grid, 256, 0, s>>>(R, Pv, N, PS, z0, n, buf, 0, nullptr, nullptr);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_unpack_planes(double2* R, double2* Pv, int npairs, size_t N, int PS, int z0, int n, const double2* buf,
                          cudaStream_t s) {
    if (n <= 0 || npairs <= 0) return;
    dim3 grid((unsigned)std::min<size_t>(((size_t)n * PS + 255) / 256, 512), npairs, 2);
    pack_planes_kernel<<<grid, 256, 0, s>>>(nullptr, nullptr, N, PS, z0, n, const_cast<double2*>(buf), 1, R, Pv);
    DOT_CUDA_TRY(cudaGetLastError());
}

}  // namespace dot
