// Jacobian contraction on FP64 tensor cores (DMMA):
//   J[b][j][i][k] = - sum_s Lam[b][j][s] U[b][i][s] G[s][k]
// (PAPER.md Eq. (Jacobian kth column), L966-972, with the sign of Eq. (2.8)).
// GEMM view: rows m = 2*(j*ls + i) + c (c = re/im of the Hadamard product
// Lam_j (.) U_i, formed in shared memory), K = |S|, N = n_p.
#include "kernels.h"

namespace dot {

namespace {

constexpr int BM = 128;      // rows per CTA (64 complex pairs)
constexpr int BN = 40;       // n_p columns per CTA (5 n8 fragments)
constexpr int BK = 16;       // support points per k-tile
constexpr int AS = BK + 4;   // padded row stride (doubles): conflict-free A fragments
constexpr int GS = BN + 4;   // padded row stride of the G tile

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) contract_kernel(int K, int ld, int ls, int n_p,
                                                       const double2* __restrict__ Lam, size_t lam_bs,
                                                       const double2* __restrict__ U, size_t u_bs,
                                                       const double* __restrict__ G, double2* J) {
    __shared__ __align__(16) double As[BM * AS];
    __shared__ __align__(16) double Gs[BK * GS];
    const int b = blockIdx.z;
    const int npairs = ld * ls;
    const int pair0 = blockIdx.x * (BM / 2);
    const int n0 = blockIdx.y * BN;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const double2* Lb = Lam + (size_t)b * lam_bs;
    const double2* Ub = U + (size_t)b * u_bs;

    double acc[2][5][2];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int ni = 0; ni < 5; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

    for (int kt = 0; kt < K; kt += BK) {
        // Hadamard-formed A tile: 64 pairs x 16 points
        for (int e = threadIdx.x; e < (BM / 2) * BK; e += blockDim.x) {
            const int lp = e / BK, kk = e % BK;
            const int pair = pair0 + lp, s = kt + kk;
            double2 v = make_double2(0.0, 0.0);
            if (pair < npairs && s < K) {
                const int j = pair / ls, i = pair - j * ls;
                v = cmul(Lb[(size_t)j * K + s], Ub[(size_t)i * K + s]);
            }
            As[(2 * lp) * AS + kk] = v.x;
            As[(2 * lp + 1) * AS + kk] = v.y;
        }
        for (int e = threadIdx.x; e < BK * BN; e += blockDim.x) {
            const int kk = e / BN, n = e % BN;
            const int s = kt + kk, col = n0 + n;
            Gs[kk * GS + n] = (s < K && col < n_p) ? G[(size_t)s * n_p + col] : 0.0;
        }
        __syncthreads();
#pragma unroll
        for (int k4 = 0; k4 < BK; k4 += 4) {
            double af[2], bf[5];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi) af[mi] = As[(warp * 16 + mi * 8 + (lane >> 2)) * AS + k4 + (lane & 3)];
#pragma unroll
            for (int ni = 0; ni < 5; ++ni) bf[ni] = Gs[(k4 + (lane & 3)) * GS + ni * 8 + (lane >> 2)];
#pragma unroll
            for (int mi = 0; mi < 2; ++mi)
#pragma unroll
                for (int ni = 0; ni < 5; ++ni) dmma(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        __syncthreads();
    }
    // epilogue: row m -> (pair, c); J[b][pair][n] complex, negated (Eq. (2.8))
    double* Jd = reinterpret_cast<double*>(J);
#pragma unroll
    for (int mi = 0; mi < 2; ++mi) {
        const int m = warp * 16 + mi * 8 + (lane >> 2);
        const int pair = pair0 + (m >> 1), c = m & 1;
        if (pair >= npairs) continue;
#pragma unroll
        for (int ni = 0; ni < 5; ++ni) {
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int col = n0 + ni * 8 + 2 * (lane & 3) + h;
                if (col < n_p) Jd[(((size_t)b * npairs + pair) * n_p + col) * 2 + c] = -acc[mi][ni][h];
            }
        }
    }
}

}  // namespace

void launch_contract(int nb, int K, int ld, int ls, int n_p, const double2* Lam, size_t lam_bstride,
                     const double2* U, size_t u_bstride, const double* G, double2* J, cudaStream_t s) {
    const int npairs = ld * ls;
    if (nb <= 0 || npairs <= 0 || n_p <= 0) return;
    if (K <= 0) {
        DOT_CUDA_TRY(cudaMemsetAsync(J, 0, (size_t)nb * npairs * n_p * sizeof(double2), s));
        return;
    }
    dim3 grid((npairs + BM / 2 - 1) / (BM / 2), (n_p + BN - 1) / BN, nb);
    contract_kernel<<<grid, 256, 0, s>>>(K, ld, ls, n_p, Lam, lam_bstride, U, u_bstride, G, J);
    DOT_CUDA_TRY(cudaGetLastError());
}

}  // namespace dot
