// Small dense helpers of the misfit / sketch algebra (PAPER.md Eq. (EsTResidual)):
// real^T x complex products (V^T R, D W, field combinations Z = U W),
// column gathers of sampled fields and deterministic sums of squares.
#include "kernels.h"

namespace dot {

namespace {

__global__ void rc_gemm_kernel(int M, int N, int K, const double* __restrict__ Rm, int ldr,
                               const double2* __restrict__ Cx, size_t sb, size_t sk, size_t sn,
                               double2* out, size_t ob, size_t om, size_t on) {
    const int b = blockIdx.z;
    const size_t total = (size_t)M * N;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const int m = (int)(e / N), n = (int)(e % N);
        const double2* c = Cx + b * sb + n * sn;
        double re = 0.0, im = 0.0;
        for (int k = 0; k < K; ++k) {
            const double r = Rm ? Rm[(size_t)k * ldr + m] : (k == m ? 1.0 : 0.0);
            const double2 v = c[k * sk];
            re = fma(r, v.x, re);
            im = fma(r, v.y, im);
        }
        out[b * ob + m * om + n * on] = make_double2(re, im);
    }
}

__global__ void gather_cols_kernel(int rows, int ncols, const double2* X, size_t xb, size_t xr,
                                   const int32_t* idx, double2* out, size_t ob, size_t orow) {
    const int b = blockIdx.z;
    const size_t total = (size_t)rows * ncols;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const int r = (int)(e / ncols), c = (int)(e % ncols);
        out[b * ob + r * orow + c] = X[b * xb + r * xr + idx[c]];
    }
}

__global__ void csub_kernel(double2* a, const double2* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        a[i] = csub(a[i], b[i]);
}

__global__ void cadd_kernel(double2* a, const double2* b, size_t n) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        a[i] = cadd(a[i], b[i]);
}

__global__ void sumsq_kernel(const double2* a, size_t n, double* out) {
    __shared__ double ws[32];
    double s = 0.0;
    for (size_t i = threadIdx.x; i < n; i += blockDim.x) s = fma(a[i].x, a[i].x, fma(a[i].y, a[i].y, s));
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) ws[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += ws[w];
        *out = t;
    }
}

// Dt[f][s][d] = D[f][d][s]
__global__ void transpose_data_kernel(const double2* D, int nf, int nd, int ns, double2* Dt) {
    const size_t total = (size_t)nf * nd * ns;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < total;
         e += (size_t)gridDim.x * blockDim.x) {
        const size_t f = e / ((size_t)nd * ns), rem = e % ((size_t)nd * ns);
        const size_t d = rem / ns, s = rem % ns;
        Dt[(f * ns + s) * nd + d] = D[e];
    }
}

// R[r][S[x]] = w[r][x]  (dense right-hand sides supported on S)
__global__ void scatter_support_kernel(double2* R, size_t N, int K, const int32_t* S, const double2* w) {
    const int r = blockIdx.y;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < K; x += gridDim.x * blockDim.x)
        R[(size_t)r * N + S[x]] = w[(size_t)r * K + x];
}

// w[f][q][x] = sum_i Z[f][i][x] sum_k C[f][q][i][k] G[x][k]
__global__ void form_support_rhs_kernel(int K, int ncol, int n_p, int nq, const double2* __restrict__ C,
                                        const double2* __restrict__ Z, const double* __restrict__ G, double2* w) {
    const int q = blockIdx.y, f = blockIdx.z;
    const double2* Cf = C + ((size_t)f * nq + q) * ncol * n_p;
    const double2* Zf = Z + (size_t)f * ncol * K;
    for (int x = blockIdx.x * blockDim.x + threadIdx.x; x < K; x += gridDim.x * blockDim.x) {
        const double* g = G + (size_t)x * n_p;
        double2 acc = make_double2(0.0, 0.0);
        for (int i = 0; i < ncol; ++i) {
            double2 c = make_double2(0.0, 0.0);
            for (int k = 0; k < n_p; ++k) {
                c.x = fma(Cf[(size_t)i * n_p + k].x, g[k], c.x);
                c.y = fma(Cf[(size_t)i * n_p + k].y, g[k], c.y);
            }
            acc = cfma(c, Zf[(size_t)i * K + x], acc);
        }
        w[((size_t)f * nq + q) * K + x] = acc;
    }
}

inline unsigned blocks_for(size_t n) {
    size_t g = (n + 255) / 256;
    return (unsigned)std::max<size_t>(1, std::min<size_t>(g, 8192));
}

__global__ void scale_cols_kernel(double2* X, size_t rows, int ncols, const double* scale) {
    const size_t tot = rows * ncols;
    for (size_t e = blockIdx.x * (size_t)blockDim.x + threadIdx.x; e < tot; e += (size_t)gridDim.x * blockDim.x) {
        const double sc = scale[e % ncols];
        X[e] = make_double2(X[e].x * sc, X[e].y * sc);
    }
}

}  // namespace

void launch_rc_gemm(int nb, int M, int N, int K, const double* Rm, int ldr, const double2* Cx,
                    size_t sb, size_t sk, size_t sn, double2* out, size_t ob, size_t om, size_t on,
                    cudaStream_t s) {
    if (nb <= 0 || M <= 0 || N <= 0) return;
    dim3 grid(blocks_for((size_t)M * N), 1, nb);
    rc_gemm_kernel<<<grid, 256, 0, s>>>(M, N, K, Rm, ldr, Cx, sb, sk, sn, out, ob, om, on);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_gather_cols(int nb, int rows, int ncols, const double2* X, size_t xb, size_t xr,
                        const int32_t* idx, double2* out, size_t ob, size_t orow, cudaStream_t s) {
    if (nb <= 0 || rows <= 0 || ncols <= 0) return;
    dim3 grid(blocks_for((size_t)rows * ncols), 1, nb);
    gather_cols_kernel<<<grid, 256, 0, s>>>(rows, ncols, X, xb, xr, idx, out, ob, orow);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_csub_inplace(double2* a, const double2* b, size_t n, cudaStream_t s) {
    if (n == 0) return;
    csub_kernel<<<blocks_for(n), 256, 0, s>>>(a, b, n);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_cadd_inplace(double2* a, const double2* b, size_t n, cudaStream_t s) {
    if (!n) return;
    cadd_kernel<<<blocks_for(n), 256, 0, s>>>(a, b, n);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_sumsq(const double2* a, size_t n, double* out, cudaStream_t s) {
    sumsq_kernel<<<1, 1024, 0, s>>>(a, n, out);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_transpose_data(const double2* D, int nf, int nd, int ns, double2* Dt, cudaStream_t s) {
    transpose_data_kernel<<<blocks_for((size_t)nf * nd * ns), 256, 0, s>>>(D, nf, nd, ns, Dt);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_scatter_support(double2* R, size_t N, int nr, const int32_t* S, int K, const double2* w, cudaStream_t s) {
    if (nr <= 0 || K <= 0) return;
    dim3 grid((unsigned)std::min((K + 255) / 256, 1024), nr);
    scatter_support_kernel<<<grid, 256, 0, s>>>(R, N, K, S, w);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_form_support_rhs(int nf, int nq, int K, int ncol, int n_p, const double2* C, const double2* Z,
                             const double* G, double2* w, cudaStream_t s) {
    if (nf <= 0 || nq <= 0 || K <= 0) return;
    dim3 grid((unsigned)std::min((K + 127) / 128, 1024), nq, nf);
    form_support_rhs_kernel<<<grid, 128, 0, s>>>(K, ncol, n_p, nq, C, Z, G, w);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_scale_cols(double2* X, size_t rows, int ncols, const double* scale, cudaStream_t s) {
    const size_t tot = rows * ncols;
    if (!tot) return;
    scale_cols_kernel<<<(unsigned)std::min<size_t>((tot + 255) / 256, 1024), 256, 0, s>>>(X, rows, ncols, scale);
    DOT_CUDA_TRY(cudaGetLastError());
}

}  // namespace dot
