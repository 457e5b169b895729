// Jacobian contraction on FP64 tensor cores (DMMA, mma.sync.m8n8k4.f64 -- on
// sm_100a the only FP64 tensor instruction; tcgen05.mma has no f64 kind):
//   J[b][j][i][k] = - sum_s Lam[b][j][s] U[b][i][s] G[s][k]
// (PAPER.md Eq. (Jacobian kth column), L966-972, with the sign of Eq. (2.8)).
// GEMM view: rows m = 2*(j*ls + i) + c (c = re/im of the Hadamard product
// Lam_j (.) U_i, formed on the fly into shared memory), reduction over the
// support K = |S|, columns n_p.
//
// CTA tile 128 rows (64 (j,i) pairs) x 8*NT columns (all parameters of a column
// block, so each Hadamard product is formed once), k-tiles of 16 support points,
// double-buffered in shared memory: the global loads of k-tile t+1 are issued
// into registers before the DMMAs of tile t and land in the other buffer after
// them -- one barrier per k-tile.  8 warps, warp w owns rows 16w .. 16w+15.
#include <array>
#include <map>
#include <mutex>

#include "arena.h"
#include "kernels.h"

namespace dot {

namespace {

constexpr int BM = 128;      // rows per CTA (64 complex pairs)
constexpr int BK = 16;       // support points per k-tile
constexpr int AS = BK + 4;   // padded row stride (doubles): conflict-free A fragments
constexpr int THREADS = 256;
constexpr int HPT = (BM / 2) * BK / THREADS;   // Hadamard products per thread per k-tile (4)

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int NT>
__global__ void __launch_bounds__(THREADS) contract_kernel(int K, int ld, int ls, int n_p,
                                                           const double2* __restrict__ Lam, size_t lam_bs,
                                                           const double2* __restrict__ U, size_t u_bs,
                                                           const double* __restrict__ G, double2* J) {
    constexpr int BN = 8 * NT;
    constexpr int GS = BN + 4;                  // padded row stride of the G tile
    constexpr int GPT = (BK * BN + THREADS - 1) / THREADS;
    extern __shared__ __align__(16) double csm[];
    // layout: A tiles [2][BM * AS], then G tiles [2][BK * GS]
    auto Abuf = [&](int bb) { return csm + bb * (BM * AS); };
    auto Gbuf = [&](int bb) { return csm + 2 * BM * AS + bb * (BK * GS); };
    const int b = blockIdx.z;
    const int npairs = ld * ls;
    const int pair0 = blockIdx.x * (BM / 2);
    const int n0 = blockIdx.y * BN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double2* Lb = Lam + (size_t)b * lam_bs;
    const double2* Ub = U + (size_t)b * u_bs;

    // per-thread Hadamard slots: element e = threadIdx.x + q*THREADS -> (lp, kk)
    const double2* lrow[HPT];
    const double2* urow[HPT];
    bool pv[HPT];
#pragma unroll
    for (int q = 0; q < HPT; ++q) {
        const int e = threadIdx.x + q * THREADS;
        const int lp = e / BK;
        const int pair = pair0 + lp;
        pv[q] = pair < npairs;
        const int j = pv[q] ? pair / ls : 0, i = pv[q] ? pair - j * ls : 0;
        lrow[q] = Lb + (size_t)j * K + (e % BK);
        urow[q] = Ub + (size_t)i * K + (e % BK);
    }
    double2 lv[HPT], uv[HPT];
    double gv[GPT];
    auto load = [&](int kt) {
#pragma unroll
        for (int q = 0; q < HPT; ++q) {
            const int s = kt + ((threadIdx.x + q * THREADS) % BK);
            const bool ok = pv[q] && s < K;
            lv[q] = ok ? lrow[q][kt] : make_double2(0.0, 0.0);
            uv[q] = ok ? urow[q][kt] : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
            const int e = threadIdx.x + q * THREADS;
            const int kk = e / BN, n = e % BN;
            const int s = kt + kk, col = n0 + n;
            gv[q] = (e < BK * BN && s < K && col < n_p) ? G[(size_t)s * n_p + col] : 0.0;
        }
    };
    auto store = [&](int buf) {
#pragma unroll
        for (int q = 0; q < HPT; ++q) {
            const int e = threadIdx.x + q * THREADS;
            const int lp = e / BK, kk = e % BK;
            const double2 v = cmul(lv[q], uv[q]);
            double* A = Abuf(buf);
            A[(2 * lp) * AS + kk] = v.x;
            A[(2 * lp + 1) * AS + kk] = v.y;
        }
#pragma unroll
        for (int q = 0; q < GPT; ++q) {
            const int e = threadIdx.x + q * THREADS;
            if (e < BK * BN) Gbuf(buf)[(e / BN) * GS + (e % BN)] = gv[q];
        }
    };

    double acc[2][NT][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    load(0);
    store(0);
    __syncthreads();
    int buf = 0;
    for (int kt = 0; kt < K; kt += BK) {
        const bool more = kt + BK < K;
        if (more) load(kt + BK);                 // global loads in flight during the DMMAs
        const double* A = Abuf(buf);
        const double* Bt = Gbuf(buf);
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double af[2], bf[NT];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = A[(warp * 16 + mi * 8 + (lane >> 2)) * AS + k4 + (lane & 3)];
#pragma unroll
            for (int ni = 0; ni < NT; ++ni) bf[ni] = Bt[(k4 + (lane & 3)) * GS + ni * 8 + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < NT; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    // epilogue: row m -> (pair, c); J[b][pair][n] complex, negated (Eq. (2.8))
    double* Jd = reinterpret_cast<double*>(J);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int m = warp * 16 + mi * 8 + (lane >> 2);
        const int pair = pair0 + (m >> 1), c = m & 1;
        if (pair >= npairs) continue;
#pragma unroll
        for (int ni = 0; ni < NT; ++ni) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = n0 + ni * 8 + 2 * (lane & 3) + h;
                if (col < n_p) Jd[(((size_t)b * npairs + pair) * n_p + col) * 2 + c] = -acc[mi][ni][h];
            }
        }
    }
}

template <int NT>
void launch_nt(int nb, int K, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride, const double2* U,
               size_t u_bstride, const double* G, double2* J, cudaStream_t s) {
    const int npairs = ld * ls;
    dim3 grid((npairs + BM / 2 - 1) / (BM / 2), (n_p + 8 * NT - 1) / (8 * NT), nb);
    const size_t smem = (size_t)(2 * BM * AS + 2 * BK * (8 * NT + 4)) * sizeof(double);
    ensure_smem(contract_kernel<NT>, smem);
    contract_kernel<NT><<<grid, THREADS, smem, s>>>(K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, J);
    DOT_CUDA_TRY(cudaGetLastError());
}

// ---------------------------------------------------------------- block-sparse
// Per basis j (grid.y) the 5 parameter columns 5j..5j+4 (one n8 fragment, 3 zero
// columns) over the support points of that basis only.  Same GEMM view and DMMA
// fragments as above; k-tiles of SBK points taken from the segment list.
constexpr int SBK = 32;
constexpr int SAS = SBK + 4;
constexpr int SGS = 8 + 4;
constexpr int SHPT = (BM / 2) * SBK / THREADS;   // Hadamard products per thread per k-tile (8)

__global__ void __launch_bounds__(THREADS) contract_sparse_kernel(int K, int ld, int ls, int n_p,
                                                                  const double2* __restrict__ Lam, size_t lam_bs,
                                                                  const double2* __restrict__ U, size_t u_bs,
                                                                  const double* __restrict__ G,
                                                                  const int32_t* __restrict__ seg,
                                                                  const int32_t* __restrict__ segoff, double2* J) {
    extern __shared__ __align__(16) double csm[];
    auto Abuf = [&](int bb) { return csm + bb * (BM * SAS); };
    auto Gbuf = [&](int bb) { return csm + 2 * BM * SAS + bb * (SBK * SGS); };
    const int b = blockIdx.z, jb = blockIdx.y;
    const int npairs = ld * ls;
    const int pair0 = blockIdx.x * (BM / 2);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double2* Lb = Lam + (size_t)b * lam_bs;
    const double2* Ub = U + (size_t)b * u_bs;
    const int s0 = segoff[jb], s1 = segoff[jb + 1];
    const int c0 = 5 * jb;

    const double2* lrow[SHPT];
    const double2* urow[SHPT];
    bool pv[SHPT];
#pragma unroll
    for (int q = 0; q < SHPT; ++q) {
        const int e = threadIdx.x + q * THREADS;
        const int pair = pair0 + e / SBK;
        pv[q] = pair < npairs;
        const int j = pv[q] ? pair / ls : 0, i = pv[q] ? pair - j * ls : 0;
        lrow[q] = Lb + (size_t)j * K;
        urow[q] = Ub + (size_t)i * K;
    }
    double2 lv[SHPT], uv[SHPT];
    double gv = 0.0;
    auto load = [&](int kt) {
#pragma unroll
        for (int q = 0; q < SHPT; ++q) {
            const int t = kt + ((threadIdx.x + q * THREADS) % SBK);
            const bool ok = pv[q] && t < s1;
            const int node = ok ? seg[t] : 0;
            lv[q] = ok ? lrow[q][node] : make_double2(0.0, 0.0);
            uv[q] = ok ? urow[q][node] : make_double2(0.0, 0.0);
        }
        {   // G tile: SBK points x 8 columns (5 used) = 256 values, one per thread
            const int kk = threadIdx.x / 8, n = threadIdx.x % 8;
            const int t = kt + kk;
            gv = (t < s1 && n < 5 && c0 + n < n_p) ? G[(size_t)seg[t] * n_p + c0 + n] : 0.0;
        }
    };
    auto store = [&](int buf) {
        double* A = Abuf(buf);
#pragma unroll
        for (int q = 0; q < SHPT; ++q) {
            const int e = threadIdx.x + q * THREADS;
            const int lp = e / SBK, kk = e % SBK;
            const double2 v = cmul(lv[q], uv[q]);
            A[(2 * lp) * SAS + kk] = v.x;
            A[(2 * lp + 1) * SAS + kk] = v.y;
        }
        Gbuf(buf)[(threadIdx.x / 8) * SGS + (threadIdx.x % 8)] = gv;
    };

    double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
    if (s0 < s1) {
        load(s0);
        store(0);
    }
    __syncthreads();
    int buf = 0;
    for (int kt = s0; kt < s1; kt += SBK) {
        const bool more = kt + SBK < s1;
        if (more) load(kt + SBK);
        const double* A = Abuf(buf);
        const double* Bt = Gbuf(buf);
#pragma unroll
        for (int k4 = 0; k4 < SBK; k4 += 4) {
            const double bf = Bt[(k4 + (lane & 3)) * SGS + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
                dmma(acc[mi][0], acc[mi][1], A[(warp * 16 + mi * 8 + (lane >> 2)) * SAS + k4 + (lane & 3)], bf);
        }
        if (more) store(buf ^ 1);
        __syncthreads();
        buf ^= 1;
    }
    double* Jd = reinterpret_cast<double*>(J);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int m = warp * 16 + mi * 8 + (lane >> 2);
        const int pair = pair0 + (m >> 1), c = m & 1;
        if (pair >= npairs) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const int n = 2 * (lane & 3) + h;
            if (n < 5 && c0 + n < n_p) Jd[(((size_t)b * npairs + pair) * n_p + c0 + n) * 2 + c] = -acc[mi][h];
        }
    }
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(valid ? 16 : 0) : "memory");
}
__device__ __forceinline__ void cp_async8(void* dst, const void* src, bool valid) {
    const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;" ::"r"(d), "l"(src), "r"(valid ? 8 : 0) : "memory");
}


__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint32_t bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(bar) : "memory");
}

// ------------------------------------- segment GEMM on pre-formed operand tiles (default)
// J[d][(q, i)] = - sum_{t in basis j} Lam[d][t] (Gs[t][q] U[i][t]) as the 3-multiply complex
// GEMM of seg_v1 above, with every FP64 ALU operation moved out of the DMMA loop: on sm_100
// DADD / DMUL issue into the FP64 pipe DMMA uses (ncu: math-pipe stalls on DADD beside DMMA,
// DMMA pipe 56-70 % with them in the loop, 100 % without, tools/dmma_probe.cu).
//  * seg_prescale_kernel writes, per frequency, the operands as blocks of 64 rows x 16
//    points (a k-tile never straddles two bases; zero rows / points pad the tails) laid out
//    exactly as the GEMM's shared stage: [64][16] double2 (re, im) then [64][16] double
//    (re + im), the point index XOR-swizzled per row so fragment loads are conflict-free
//    (double2: kk ^ 4 (row & 1); double: kk ^ 4 (row & 3)).  A rows are detectors (Lam),
//    B rows are (q, i) = q ls + i with the weight folded in (Gs[t][q] U[i][t]).
//  * seg_tma_gemm_kernel: one producer lane streams the A and B block of each k-tile with one
//    cp.async.bulk each into a 4-stage ring (full / empty mbarriers); 8 consumer warps (2 per
//    scheduler), warp tile 16 x 32, run LDS + DMMA only (3 DMMA per fragment pair).
constexpr int kMaxRbf = 256;                           // bases of one problem (segment GEMM tables)
namespace tma {
constexpr int QM = 64, KT = 16, BLK = QM * KT * 24, NST = 4, NCW = 8, NT = 32 * (NCW + 1);
constexpr size_t SMEM = 128 + (size_t)NST * 2 * BLK;
static_assert(SMEM <= 232448, "seg_tma_gemm shared memory");
}  // namespace tma

// Blocks [0, nA) of grid.y: A side (detector rows of Lam), blocks [nA, ..): B side rows
// (q, i) = q ls + i of column tiles rtB0 + (y - nA), weights folded in.
__global__ void __launch_bounds__(256) seg_prescale_kernel(int ld, int ls, int T, const double2* __restrict__ Lam,
                                                           const double2* __restrict__ U,
                                                           const double* __restrict__ Gs,
                                                           const int4* __restrict__ ktile, int KTn, int nA, int rtB0,
                                                           unsigned char* outA, unsigned char* outB) {
    const int g = blockIdx.x;
    const bool bside = (int)blockIdx.y >= nA;
    const int rt = bside ? rtB0 + (int)blockIdx.y - nA : (int)blockIdx.y;
    unsigned char* base = bside ? outB + ((size_t)(blockIdx.y - nA) * KTn + g) * tma::BLK
                                : outA + ((size_t)blockIdx.y * KTn + g) * tma::BLK;
    double2* o2 = reinterpret_cast<double2*>(base);
    double* o1 = reinterpret_cast<double*>(base + tma::QM * tma::KT * 16);
    __shared__ int rowq[tma::QM], rowi[tma::QM];
    if (threadIdx.x < tma::QM) {                 // row -> (q, i) once per block (no per-element divide)
        const int n = rt * tma::QM + threadIdx.x;
        const int q = bside ? n / ls : 0;
        rowq[threadIdx.x] = q;
        rowi[threadIdx.x] = bside ? n - q * ls : n;
    }
    __syncthreads();
    const int4 kt = ktile[g];
    const int rows = bside ? 5 * ls : ld;
    for (int e = threadIdx.x; e < tma::QM * tma::KT; e += blockDim.x) {
        const int r = e >> 4, kk = e & 15, n = rt * tma::QM + r, t = kt.x + kk;
        double2 v = make_double2(0.0, 0.0);
        double sm = 0.0;
        if (n < rows && t < kt.y) {
            if (!bside) {
                v = Lam[(size_t)n * T + t];
                sm = v.x + v.y;
            } else {
                const double2 u = U[(size_t)rowi[r] * T + t];
                const double w = Gs[(size_t)t * 5 + rowq[r]];
                v = make_double2(w * u.x, w * u.y);
                sm = w * (u.x + u.y);
            }
        }
        // streaming stores: the blocks of the next frequency must not evict the operands the
        // concurrent GEMM of the current frequency re-reads from L2
        __stcs(o2 + r * 16 + (kk ^ ((r & 1) << 2)), v);
        __stcs(o1 + r * 16 + (kk ^ ((r & 3) << 2)), sm);
    }
}

// Persistent, dynamically scheduled: the producer lane claims work items from a global
// counter (items ordered basis jorder[.] largest first, then column tile, then detector tile:
// longest-first list scheduling) and streams their k-tiles back to back through the ring,
// tagging each stage with (item, k-tile, k-tiles of the item); the next item's first tiles
// land during the current item's last DMMAs and epilogue.  An item of a basis without points
// is a stage with no data (its J block is written as zeros); item -1 ends the CTA.
__global__ void __launch_bounds__(tma::NT, 1) seg_tma_gemm_kernel(int ld, int ls, int n_p, const unsigned char* Ap,
                                                                 const unsigned char* Bp, int KTn,
                                                                 const int32_t* __restrict__ kto,
                                                                 const int32_t* __restrict__ jorder, int nDT, int nn,
                                                                 int nitems, int nt0, int* counter, double2* J) {
    using tma::BLK;
    using tma::KT;
    using tma::NCW;
    using tma::NST;
    constexpr int TM = tma::QM;
    extern __shared__ __align__(128) unsigned char tsm[];
    const uint32_t bar0 = static_cast<uint32_t>(__cvta_generic_to_shared(tsm));   // full[NST], empty[NST]
    int* meta = reinterpret_cast<int*>(tsm + 16 * NST);                             // [NST][4]
    const uint32_t st0 = bar0 + 128;
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int per_j = nDT * nn;
    __shared__ int s_jorder[kMaxRbf], s_kto[kMaxRbf + 1];
    const int nrbf = nitems / per_j;
    for (int i = tid; i <= nrbf; i += blockDim.x) {
        s_kto[i] = kto[i];
        if (i < nrbf) s_jorder[i] = jorder[i];
    }
    if (tid == 0) {
        for (int s = 0; s < NST; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar0 + 8 * s), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar0 + 8 * (NST + s)), "r"(32 * NCW));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NCW) {                                   // producer: one lane claims items, streams blocks
        if (lane == 0) {
            uint32_t gt = 0;
            // stage tag: (t, k-tiles of the item, basis j, tile = dt + nDT ntl); j = -1 ends the CTA
            auto stage = [&](int t, int nkt, int j, int tile, const unsigned char* a, const unsigned char* b) {
                const uint32_t s = gt % NST;
                if (gt >= NST) mbar_wait(bar0 + 8 * (NST + s), ((gt / NST) - 1) & 1);
                meta[4 * s] = t;
                meta[4 * s + 1] = nkt;
                meta[4 * s + 2] = j;
                meta[4 * s + 3] = tile;
                const uint32_t fb = bar0 + 8 * s, dA = st0 + s * 2 * BLK;
                if (a) {
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(fb), "r"(2 * BLK)
                                 : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dA),
                        "l"(a), "r"(BLK), "r"(fb)
                        : "memory");
                    asm volatile(
                        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                            dA + BLK),
                        "l"(b), "r"(BLK), "r"(fb)
                        : "memory");
                } else {
                    mbar_arrive(fb);
                }
                ++gt;
            };
            // (claiming the next item one ahead measured slower: 1.15 vs 1.01 ms at full64)
            for (;;) {
                const int it = atomicAdd(counter, 1);
                if (it >= nitems) {
                    stage(0, 0, -1, 0, nullptr, nullptr);
                    break;
                }
                const int jj = it / per_j, r = it % per_j, ntl = r / nDT, dt = r % nDT;
                const int j = s_jorder[jj];
                const int g0 = s_kto[j], nkt = s_kto[j + 1] - g0;
                const unsigned char* a = Ap + ((size_t)dt * KTn + g0) * BLK;
                const unsigned char* b = Bp + ((size_t)ntl * KTn + g0) * BLK;
                if (nkt == 0) stage(0, 0, j, r, nullptr, nullptr);
                for (int t = 0; t < nkt; ++t) stage(t, nkt, j, r, a + (size_t)t * BLK, b + (size_t)t * BLK);
            }
        }
        return;
    }
    const int wm = (warp & 3) * 16, wn = (warp >> 2) * 32;
    const int r4 = lane >> 2, sw2 = (r4 & 1) << 2, sw1 = (r4 & 3) << 2;
    double p1[2][4][2], p2[2][4][2], p3[2][4][2];
    for (uint32_t gt = 0;; ++gt) {
        const uint32_t s = gt % NST;
        mbar_wait(bar0 + 8 * s, (gt / NST) & 1);
        const int t = meta[4 * s], nkt = meta[4 * s + 1], j = meta[4 * s + 2], tile = meta[4 * s + 3];
        if (j < 0) break;
        if (t == 0) {
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                    for (int h = 0; h < 2; ++h) p1[mi][ni][h] = p2[mi][ni][h] = p3[mi][ni][h] = 0.0;
        }
        if (nkt > 0) {
            const unsigned char* sa = tsm + 128 + (size_t)s * 2 * BLK;
            const double2* A2 = reinterpret_cast<const double2*>(sa);
            const double* A1 = reinterpret_cast<const double*>(sa + TM * KT * 16);
            const double2* B2 = reinterpret_cast<const double2*>(sa + BLK);
            const double* B1 = reinterpret_cast<const double*>(sa + BLK + TM * KT * 16);
#pragma unroll
            for (int k4 = 0; k4 < KT; k4 += 4) {
                const int kk = k4 + (lane & 3);
                double2 a[2];
                double as[2];
#pragma unroll
                for (int mi = 0; mi < 2; ++mi) {
                    const int rr = wm + mi * 8 + r4;
                    a[mi] = A2[rr * 16 + (kk ^ sw2)];
                    as[mi] = A1[rr * 16 + (kk ^ sw1)];
                }
#pragma unroll
                for (int ni = 0; ni < 4; ++ni) {
                    const int rr = wn + ni * 8 + r4;
                    const double2 b = B2[rr * 16 + (kk ^ sw2)];
                    const double bs = B1[rr * 16 + (kk ^ sw1)];
#pragma unroll
                    for (int mi = 0; mi < 2; ++mi) {
                        dmma(p1[mi][ni][0], p1[mi][ni][1], a[mi].x, b.x);
                        dmma(p2[mi][ni][0], p2[mi][ni][1], a[mi].y, b.y);
                        dmma(p3[mi][ni][0], p3[mi][ni][1], as[mi], bs);
                    }
                }
            }
        }
        mbar_arrive(bar0 + 8 * (NST + s));
        if (t + 1 < nkt) continue;
        // last k-tile of the item: epilogue J[(d, i)][5 j + q] = -C[d][q ls + i]
        const int ntl = tile / nDT, dt = tile - ntl * nDT;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi) {
            const int d = dt * TM + wm + mi * 8 + r4;
            if (d >= ld) continue;
#pragma unroll
            for (int ni = 0; ni < 4; ++ni)
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const int n = (nt0 + ntl) * TM + wn + ni * 8 + 2 * (lane & 3) + h;
                    if (n >= 5 * ls) continue;
                    const int q = n / ls, i = n - q * ls;
                    const double re = p1[mi][ni][h] - p2[mi][ni][h];
                    const double im = p3[mi][ni][h] - p1[mi][ni][h] - p2[mi][ni][h];
                    J[((size_t)d * ls + i) * n_p + 5 * j + q] = make_double2(-re, -im);
                }
        }
    }
}

// ---------------------------------------------- small panels: split over the k-tiles
// The sketched and optimized-direction contractions have ld x ls <= 256 pairs (12 x 12 at
// the BASELINE configs): a GEMM tile would be mostly padding and 16 bases x n_freq tiles
// cannot fill 148 SMs.  One CTA per (basis j, chunk of SMALL_KC k-tiles of that basis,
// frequency) accumulates all ld x ls x 5 outputs of the basis over the chunk's points (FP64
// FMA on shared-memory copies of the fields, one k-tile at a time); a second kernel adds the
// chunks of each basis in chunk order (deterministic, no atomics) into J.
constexpr int SMALL_PAIRS = 256, SMALL_ROWS = 160;   // ld * ls and ld + ls limits of the small form
constexpr int SMALL_KC = 4;                          // k-tiles per CTA

__global__ void __launch_bounds__(256) contract_small_kernel(int K, int ld, int ls, int n_p,
                                                             const double2* __restrict__ Lam, size_t lam_bs,
                                                             const double2* __restrict__ U, size_t u_bs,
                                                             const double* __restrict__ G,
                                                             const int32_t* __restrict__ seg,
                                                             const int4* __restrict__ ktile,
                                                             const int32_t* __restrict__ kto, int nch,
                                                             double2* __restrict__ part) {
    __shared__ double2 sf[SMALL_ROWS][16];                 // rows [0, ld): Lam, [ld, ld + ls): U
    __shared__ double sg[16][5];
    const int j = blockIdx.x, c = blockIdx.y, f = blockIdx.z;
    const int g0 = kto[j] + c * SMALL_KC, g1 = min(g0 + SMALL_KC, kto[j + 1]);
    const int nout = ld * ls * 5;
    double2* out = part + (((size_t)f * gridDim.x + j) * nch + c) * nout;
    if (g0 >= g1) {                                        // past this basis's k-tiles: zero chunk
        for (int o = threadIdx.x; o < nout; o += blockDim.x) out[o] = make_double2(0.0, 0.0);
        return;
    }
    const double2* Lf = Lam + (size_t)f * lam_bs;
    const double2* Uf = U + (size_t)f * u_bs;
    constexpr int PER = 8;                                 // outputs per thread kept in registers
    double re[PER], im[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) re[u] = im[u] = 0.0;
    for (int g = g0; g < g1; ++g) {
        const int4 kt = ktile[g];
        const int np = min(16, kt.y - kt.x);
        __syncthreads();                                   // previous tile consumed
        for (int e = threadIdx.x; e < (ld + ls) * 16; e += blockDim.x) {
            const int r = e >> 4, t = e & 15;
            double2 v = make_double2(0.0, 0.0);
            if (t < np) {
                const int node = seg[kt.x + t];
                v = r < ld ? Lf[(size_t)r * K + node] : Uf[(size_t)(r - ld) * K + node];
            }
            sf[r][t] = v;
        }
        if (threadIdx.x < 80) {
            const int t = threadIdx.x / 5, q = threadIdx.x % 5;
            sg[t][q] = t < np ? G[(size_t)seg[kt.x + t] * n_p + 5 * j + q] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int u = 0; u < PER; ++u) {
            const int o = threadIdx.x + u * blockDim.x;
            if (o >= nout) break;
            const int q = o % 5, pr = o / 5, d = pr / ls, i = pr - d * ls;
#pragma unroll
            for (int t = 0; t < 16; ++t) {
                const double2 h = cmul(sf[d][t], sf[ld + i][t]);
                re[u] = fma(h.x, sg[t][q], re[u]);
                im[u] = fma(h.y, sg[t][q], im[u]);
            }
        }
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
        const int o = threadIdx.x + u * blockDim.x;
        if (o < nout) out[o] = make_double2(re[u], im[u]);
    }
}

// J[f][pair][5 j + q] = - sum_c part[f][j][c][pair * 5 + q]   (grid: outputs, bases, frequencies)
__global__ void contract_small_reduce_kernel(int ls, int n_p, int nout, int nch, const double2* __restrict__ part,
                                             double2* J) {
    const int j = blockIdx.y, f = blockIdx.z;
    const int o = blockIdx.x * blockDim.x + threadIdx.x;
    if (o >= nout) return;
    const double2* p = part + ((size_t)f * gridDim.y + j) * nch * nout + o;
    double re = 0.0, im = 0.0;
    for (int c = 0; c < nch; ++c) {
        const double2 v = p[(size_t)c * nout];
        re += v.x;
        im += v.y;
    }
    const int pr = o / 5, q = o % 5;
    J[((size_t)f * (nout / 5) + pr) * n_p + 5 * j + q] = make_double2(-re, -im);
}

// Gs[t][q] = G[seg[t]][5 j + q] for the points t of basis j (basis-ordered weights)
__global__ void seg_weights_kernel(const double* __restrict__ G, int n_p, const int32_t* seg, const int32_t* segoff,
                                   double* Gs) {
    const int j = blockIdx.y;
    for (int t = segoff[j] + blockIdx.x * blockDim.x + threadIdx.x; t < segoff[j + 1]; t += gridDim.x * blockDim.x)
        for (int q = 0; q < 5; ++q) Gs[(size_t)t * 5 + q] = 5 * j + q < n_p ? G[(size_t)seg[t] * n_p + 5 * j + q] : 0.0;
}

// idx[t] = slot[seg[t]]
__global__ void compose_index_kernel(const int32_t* seg, int T, const int32_t* slot, int32_t* idx) {
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < T; t += gridDim.x * blockDim.x) idx[t] = slot[seg[t]];
}

__global__ void rbf_flags_kernel(const double* __restrict__ G, int K, int n_p, int n_rbf, int32_t* F) {
    const size_t tot = (size_t)K * n_rbf;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const int j = (int)(e / K), s = (int)(e % K);
        bool nz = false;
        for (int q = 0; q < 5 && 5 * j + q < n_p; ++q) nz |= G[(size_t)s * n_p + 5 * j + q] != 0.0;
        F[e] = nz ? 1 : 0;
    }
}

__global__ void rbf_segments_kernel(const int32_t* F, const int32_t* pos, int K, int n_rbf, const int32_t* total,
                                    int32_t* seg, int32_t* off) {
    const size_t tot = (size_t)K * n_rbf;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        if (F[e]) seg[pos[e]] = (int32_t)(e % K);
        if (e % K == 0) off[e / K] = pos[e];
    }
    if (blockIdx.x == 0 && threadIdx.x == 0) off[n_rbf] = *total;
}

}  // namespace

void launch_rbf_flags(const double* G, int K, int n_rbf, int32_t* F, cudaStream_t s) {
    const size_t tot = (size_t)K * n_rbf;
    if (!tot) return;
    rbf_flags_kernel<<<(unsigned)std::min<size_t>((tot + 255) / 256, 8192), 256, 0, s>>>(G, K, 5 * n_rbf, n_rbf, F);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_rbf_segments(const int32_t* F, const int32_t* pos, int K, int n_rbf, const int32_t* total, int32_t* seg,
                         int32_t* off, cudaStream_t s) {
    const size_t tot = (size_t)K * n_rbf;
    rbf_segments_kernel<<<(unsigned)std::max<size_t>(1, std::min<size_t>((tot + 255) / 256, 8192)), 256, 0, s>>>(
        F, pos, K, n_rbf, total, seg, off);
    DOT_CUDA_TRY(cudaGetLastError());
}

bool contract_seg_applies(int ld, int ls, const GSparse* sp, int n_p) {
    return sp && sp->seg && sp->n_rbf * 5 == n_p && sp->n_rbf <= kMaxRbf && ld >= 32 && ls >= 8;
}


void launch_seg_weights(const double* G, int n_p, const GSparse& sp, double* Gs, cudaStream_t s) {
    if (sp.total <= 0) return;
    seg_weights_kernel<<<dim3(32, sp.n_rbf), 256, 0, s>>>(G, n_p, sp.seg, sp.segoff, Gs);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_compose_index(const int32_t* seg, int T, const int32_t* slot, int32_t* idx, cudaStream_t s) {
    if (T <= 0) return;
    compose_index_kernel<<<(unsigned)std::min(1024, (T + 255) / 256), 256, 0, s>>>(seg, T, slot, idx);
    DOT_CUDA_TRY(cudaGetLastError());
}

size_t contract_seg_tma_bytes(int ld, int ls, long long total, int n_rbf) {
    const size_t kts = (size_t)(total + tma::KT - 1) / tma::KT + n_rbf;
    return ((size_t)(ld + tma::QM - 1) / tma::QM + (5 * (size_t)ls + tma::QM - 1) / tma::QM) * kts * tma::BLK;
}

// Side stream of the current device for the operand prescale (created once, non-blocking).
static cudaStream_t prescale_stream() {
    static std::mutex mtx;
    static std::map<int, cudaStream_t> streams;
    int dev = 0;
    DOT_CUDA_TRY(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lock(mtx);
    auto it = streams.find(dev);
    if (it != streams.end()) return it->second;
    cudaStream_t st = nullptr;
    DOT_CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    streams[dev] = st;
    return st;
}

void contract_seg_tma(int nb, int T, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                      const double2* U, size_t u_bstride, const double* Gs, const GSparse& sp, double2* J,
                      Arena& arena, cudaStream_t s, int64_t* launches, double* dmma_flops) {
    if (nb <= 0 || ld <= 0 || ls <= 0) return;
    const int npairs = ld * ls;
    if (T <= 0 || sp.ktiles <= 0) {
        DOT_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)nb * npairs * n_p * sizeof(double2), s));
        return;
    }
    const int KTn = sp.ktiles;
    if (sp.n_rbf > kMaxRbf) throw Error(DOT_ERR_ARG, "segment GEMM supports up to 256 bases");
    const int nDT = (ld + tma::QM - 1) / tma::QM, nNT = (5 * ls + tma::QM - 1) / tma::QM;
    const size_t per_tile = (size_t)KTn * tma::BLK;
    const size_t set_bytes = (size_t)(nDT + nNT) * per_tile;       // one frequency's A and B tiles
    // executed DMMA flops: per (item, k-tile) 3 products of 64 x 64 x 16 real multiply-adds
    if (dmma_flops) *dmma_flops += (double)nb * KTn * nDT * nNT * 3.0 * 2.0 * tma::QM * tma::QM * tma::KT;
    ensure_smem(seg_tma_gemm_kernel, tma::SMEM);
    int sms = 0, dev = 0;
    DOT_CUDA_TRY(cudaGetDevice(&dev));
    DOT_CUDA_TRY(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    auto gemm = [&](int f, const unsigned char* A, const unsigned char* B, int nt0, int nn, int* counter) {
        const int nitems = sp.n_rbf * nDT * nn;
        seg_tma_gemm_kernel<<<std::min(nitems, sms), tma::NT, tma::SMEM, s>>>(
            ld, ls, n_p, A, B, KTn, sp.kto, sp.jorder, nDT, nn, nitems, nt0, counter, J + (size_t)f * npairs * n_p);
        DOT_CUDA_TRY(cudaGetLastError());
    };
    auto prescale = [&](int f, unsigned char* A, unsigned char* B, int nA, int nt0, int nn, cudaStream_t st) {
        seg_prescale_kernel<<<dim3(KTn, nA + nn), 256, 0, st>>>(ld, ls, T, Lam + (size_t)f * lam_bstride,
                                                               U + (size_t)f * u_bstride, Gs, sp.ktile, KTn, nA, nt0,
                                                               A, B);
        DOT_CUDA_TRY(cudaGetLastError());
    };
    const bool chunk_env = std::getenv("DOT_SEG_CHUNK") != nullptr;       // tests: force the chunked path
    if (nb > 1 && !chunk_env && arena.largest_free() >= 2 * set_bytes + (64u << 20)) {
        // two operand sets: the prescale of frequency f+1 (memory-bound, side stream) runs while
        // the GEMM of frequency f (DMMA-bound) owns the SMs' tensor pipes
        DBuf<unsigned char> buf[2] = {DBuf<unsigned char>(arena, set_bytes), DBuf<unsigned char>(arena, set_bytes)};
        DBuf<int> counters(arena, nb);
        DOT_CUDA_TRY(cudaMemsetAsync(counters.get(), 0, nb * sizeof(int), s));
        cudaStream_t s2 = prescale_stream();
        // events of this host thread and device, created once (calls of one thread are ordered)
        static thread_local std::map<int, std::array<cudaEvent_t, 5>> evs;
        auto evit = evs.find(dev);
        if (evit == evs.end()) {
            std::array<cudaEvent_t, 5> e5;
            for (auto& e : e5) DOT_CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
            evit = evs.emplace(dev, e5).first;
        }
        cudaEvent_t* ev = evit->second.data();
        cudaEvent_t &in_ready = ev[0], *pre = ev + 1, *used = ev + 3;
        DOT_CUDA_TRY(cudaEventRecord(in_ready, s));
        DOT_CUDA_TRY(cudaStreamWaitEvent(s2, in_ready, 0));
        for (int f = 0; f < nb; ++f) {
            const int b = f & 1;
            unsigned char* A = buf[b].get();
            unsigned char* B = A + (size_t)nDT * per_tile;
            if (f >= 2) DOT_CUDA_TRY(cudaStreamWaitEvent(s2, used[b], 0));     // GEMM f-2 done with buf b
            prescale(f, A, B, nDT, 0, nNT, s2);
            DOT_CUDA_TRY(cudaEventRecord(pre[b], s2));
            DOT_CUDA_TRY(cudaStreamWaitEvent(s, pre[b], 0));
            gemm(f, A, B, 0, nNT, counters.get() + f);
            DOT_CUDA_TRY(cudaEventRecord(used[b], s));
            *launches += 2;
        }
        return;
    }
    // one operand set; B tiles of a frequency in chunks of column tiles when the workspace is short
    DBuf<unsigned char> Ap(arena, nDT * per_tile);
    const size_t room = arena.largest_free(), margin = (size_t)1 << 20;     // margin: the counters
    int chunk = (int)std::max<size_t>(1, std::min<size_t>(nNT, room > per_tile + margin ? (room - margin) / per_tile : 1));
    if (chunk_env) chunk = std::max(1, std::min(chunk, std::atoi(std::getenv("DOT_SEG_CHUNK"))));
    DBuf<unsigned char> Bp(arena, (size_t)chunk * per_tile);
    const int nch = (nNT + chunk - 1) / chunk;
    DBuf<int> counters(arena, (size_t)nb * nch);
    DOT_CUDA_TRY(cudaMemsetAsync(counters.get(), 0, (size_t)nb * nch * sizeof(int), s));
    for (int f = 0; f < nb; ++f) {
        for (int nt0 = 0; nt0 < nNT; nt0 += chunk) {
            const int nn = std::min(chunk, nNT - nt0);
            prescale(f, Ap.get(), Bp.get(), nt0 == 0 ? nDT : 0, nt0, nn, s);   // A tiles once per frequency
            gemm(f, Ap.get(), Bp.get(), nt0, nn, counters.get() + f * nch + nt0 / chunk);
            *launches += 2;
        }
    }
}

void launch_contract(int nb, int K, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                     const double2* U, size_t u_bstride, const double* G, double2* J, cudaStream_t s,
                     const GSparse* sp, Arena* arena, int64_t* launches) {
    const int npairs = ld * ls;
    if (nb <= 0 || npairs <= 0 || n_p <= 0) return;
    if (K <= 0) {
        DOT_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)nb * npairs * n_p * sizeof(double2), s));
        return;
    }
    if (sp && sp->seg && sp->ktile && sp->n_rbf * 5 == n_p && arena && npairs <= SMALL_PAIRS && ld + ls <= SMALL_ROWS) {
        if (sp->ktiles == 0) {
            DOT_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)nb * npairs * n_p * sizeof(double2), s));
            return;
        }
        const int nch = (sp->maxkt + SMALL_KC - 1) / SMALL_KC, nout = npairs * 5;
        DBuf<double2> part(*arena, (size_t)nb * sp->n_rbf * nch * nout);
        contract_small_kernel<<<dim3(sp->n_rbf, nch, nb), 256, 0, s>>>(K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride,
                                                                      G, sp->seg, sp->ktile, sp->kto, nch, part.get());
        DOT_CUDA_TRY(cudaGetLastError());
        contract_small_reduce_kernel<<<dim3((nout + 127) / 128, sp->n_rbf, nb), 128, 0, s>>>(ls, n_p, nout, nch,
                                                                                           part.get(), J);
        DOT_CUDA_TRY(cudaGetLastError());
        if (launches) *launches += 2;
        return;
    }
    if (launches) *launches += 1;
    if (sp && sp->seg && sp->n_rbf * 5 == n_p) {
        dim3 grid((npairs + BM / 2 - 1) / (BM / 2), sp->n_rbf, nb);
        const size_t smem = (size_t)(2 * BM * SAS + 2 * SBK * SGS) * sizeof(double);
        ensure_smem(contract_sparse_kernel, smem);
        contract_sparse_kernel<<<grid, THREADS, smem, s>>>(K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, sp->seg,
                                                           sp->segoff, J);
        DOT_CUDA_TRY(cudaGetLastError());
        return;
    }
    // all parameters of a column block in one CTA (one Hadamard formation per pair)
    if (n_p <= 24) launch_nt<3>(nb, K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, J, s);
    else if (n_p <= 40) launch_nt<5>(nb, K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, J, s);
    else launch_nt<10>(nb, K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, J, s);
}

}  // namespace dot
