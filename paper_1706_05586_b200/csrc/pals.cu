// PaLS absorption mu(x, p) (Eqs. (2.3)-(2.4)), the support S of
// dA/dp (L972 "we first find the few nonzero components of dA/dp_k"), the
// Jacobian weights G = theta dmu/dp on S, and the compaction machinery that
// builds the sample set P = S u detectors.
#include "kernels.h"

namespace dot {

namespace {

__device__ __forceinline__ double wendland(double r) {       // (1-r)_+^4 (4r+1), reading R7
    if (r >= 1.0) return 0.0;
    double a = 1.0 - r, a2 = a * a;
    return a2 * a2 * (4.0 * r + 1.0);
}
__device__ __forceinline__ double wendland_d(double r) {     // -20 r (1-r)_+^3
    if (r >= 1.0) return 0.0;
    double a = 1.0 - r;
    return -20.0 * r * a * a * a;
}
__device__ __forceinline__ double heaviside(double t, double eps) {    // reading R8
    if (t < -eps) return 0.0;
    if (t > eps) return 1.0;
    return 0.5 * (1.0 + t / eps + sin(M_PI * t / eps) / M_PI);
}
__device__ __forceinline__ double heaviside_d(double t, double eps) {
    if (fabs(t) > eps) return 0.0;
    return (1.0 + cos(M_PI * t / eps)) / (2.0 * eps);
}

__device__ __forceinline__ void node_xyz(const PalsConst& c, int n, double& x, double& y, double& z,
                                         int& k) {
    int i = n % c.nx, j = (n / c.nx) % c.ny;
    k = n / (c.nx * c.ny);
    x = (i + 1) * c.hx;
    y = (j + 1) * c.hy;
    z = k * c.hz;
}

__device__ double pals_phi(const PalsConst& c, const double* p, double x, double y, double z) {
    double phi = 0.0;
    for (int b = 0; b < c.n_rbf; ++b) {
        const double al = p[5 * b], be = p[5 * b + 1];
        const double dx = x - p[5 * b + 2], dy = y - p[5 * b + 3], dz = z - p[5 * b + 4];
        const double r = sqrt(be * be * (dx * dx + dy * dy + dz * dz) + c.gamma * c.gamma);
        phi += al * wendland(r);
    }
    return phi;
}

__global__ void pals_eval_kernel(PalsConst c, const double* __restrict__ params, double* mu,
                                 int32_t* flagS, int32_t* flagP) {
    extern __shared__ double sp[];
    for (int i = threadIdx.x; i < 5 * c.n_rbf; i += blockDim.x) sp[i] = params[i];
    __syncthreads();
    const int N = c.nx * c.ny * c.nz;
    for (int n = blockIdx.x * blockDim.x + threadIdx.x; n < N; n += gridDim.x * blockDim.x) {
        double x, y, z;
        int k;
        node_xyz(c, n, x, y, z, k);
        const double t = pals_phi(c, sp, x, y, z) - c.cutoff;
        const double H = heaviside(t, c.eps);
        mu[n] = c.mua_in * H + c.mua_out * (1.0 - H);
        const int s = heaviside_d(t, c.eps) != 0.0 ? 1 : 0;
        flagS[n] = s;
        flagP[n] = s;
    }
}

__global__ void mark_nodes_kernel(int32_t* flag, const int32_t* nodes, int n) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) flag[nodes[a]] = 1;
}

// ---- three-phase exclusive scan (block sums -> scan of sums -> add)
constexpr int kScanBlock = 1024;

__global__ void scan_block_kernel(const int32_t* in, int32_t* out, size_t n, int32_t* bsum) {
    __shared__ int32_t wsum[32];
    const size_t i = blockIdx.x * (size_t)kScanBlock + threadIdx.x;
    const int v = i < n ? in[i] : 0;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
        int s = wsum[lane];
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, s, o);
            if (lane >= o) s += y;
        }
        wsum[lane] = s;
    }
    __syncthreads();
    const int incl = x + (w > 0 ? wsum[w - 1] : 0);
    if (i < n) out[i] = incl - v;
    if (threadIdx.x == kScanBlock - 1) bsum[blockIdx.x] = incl;
}

__global__ void scan_sums_kernel(int32_t* bsum, int nb, int32_t* total) {
    // single block, sequential chunks of 1024
    __shared__ int32_t carry;
    __shared__ int32_t wsum[32];
    if (threadIdx.x == 0) carry = 0;
    __syncthreads();
    for (int base = 0; base < nb; base += kScanBlock) {
        const int i = base + threadIdx.x;
        const int v = i < nb ? bsum[i] : 0;
        const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
        int x = v;
        for (int o = 1; o < 32; o <<= 1) {
            int y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
        }
        if (lane == 31) wsum[w] = x;
        __syncthreads();
        if (w == 0) {
            int s = wsum[lane];
            for (int o = 1; o < 32; o <<= 1) {
                int y = __shfl_up_sync(0xffffffffu, s, o);
                if (lane >= o) s += y;
            }
            wsum[lane] = s;
        }
        __syncthreads();
        const int incl = x + (w > 0 ? wsum[w - 1] : 0);
        const int c0 = carry;
        if (i < nb) bsum[i] = c0 + incl - v;
        __syncthreads();
        if (threadIdx.x == kScanBlock - 1) carry = c0 + incl;
        __syncthreads();
    }
    if (threadIdx.x == 0) *total = carry;
}

__global__ void scan_add_kernel(int32_t* out, size_t n, const int32_t* bsum) {
    const size_t i = blockIdx.x * (size_t)kScanBlock + threadIdx.x;
    if (i < n) out[i] += bsum[blockIdx.x];
}

__global__ void compact_kernel(const int32_t* flag, const int32_t* pos, size_t n, int32_t* out) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        if (flag[i]) out[pos[i]] = (int32_t)i;
}

__global__ void gather_rank_kernel(const int32_t* pos, const int32_t* nodes, int n, int32_t* out) {
    for (int a = blockIdx.x * blockDim.x + threadIdx.x; a < n; a += gridDim.x * blockDim.x) out[a] = pos[nodes[a]];
}

// G[s][k] = theta(z) dmu/dp_k at node S[s]; chain rule of Eqs. (2.3)-(2.4).
__global__ void pals_grad_kernel(PalsConst c, const double* __restrict__ params, const int32_t* S, int K,
                                 double* G) {
    extern __shared__ double sp[];
    for (int i = threadIdx.x; i < 5 * c.n_rbf; i += blockDim.x) sp[i] = params[i];
    __syncthreads();
    const int np = 5 * c.n_rbf;
    for (int s = blockIdx.x * blockDim.x + threadIdx.x; s < K; s += gridDim.x * blockDim.x) {
        double x, y, z;
        int k;
        node_xyz(c, S[s], x, y, z, k);
        const double th = (k == 0 || k == c.nz - 1) ? 0.5 : 1.0;
        const double t = pals_phi(c, sp, x, y, z) - c.cutoff;
        const double w = th * (c.mua_in - c.mua_out) * heaviside_d(t, c.eps);
        double* g = G + (size_t)s * np;
        for (int b = 0; b < c.n_rbf; ++b) {
            const double al = sp[5 * b], be = sp[5 * b + 1];
            const double dx = x - sp[5 * b + 2], dy = y - sp[5 * b + 3], dz = z - sp[5 * b + 4];
            const double d2 = dx * dx + dy * dy + dz * dz;
            const double r = sqrt(be * be * d2 + c.gamma * c.gamma);
            const double ps = wendland(r), dps = wendland_d(r);
            const double f = w * al * dps / r;
            g[5 * b + 0] = w * ps;
            g[5 * b + 1] = f * be * d2;
            g[5 * b + 2] = -f * be * be * dx;
            g[5 * b + 3] = -f * be * be * dy;
            g[5 * b + 4] = -f * be * be * dz;
        }
    }
}

// off[z*ntiles + t] = first sample with node >= (z*ny + t*TY)*nx ; off[nz*ntiles] = nP
__global__ void sample_offsets_kernel(const int32_t* P, int nP, int nx, int ny, int nz, int TY,
                                      int ntiles, int32_t* off) {
    const int total = nz * ntiles;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e <= total; e += gridDim.x * blockDim.x) {
        if (e == total) {
            off[e] = nP;
            continue;
        }
        const int z = e / ntiles, t = e % ntiles;
        const long long key = ((long long)z * ny + (long long)t * TY) * nx;
        int lo = 0, hi = nP;
        while (lo < hi) {
            int mid = (lo + hi) >> 1;
            if ((long long)P[mid] < key) lo = mid + 1;
            else hi = mid;
        }
        off[e] = lo;
    }
}

inline unsigned grid_for(size_t n, int bs, unsigned cap = 65535u * 4) {
    size_t g = (n + bs - 1) / bs;
    if (g < 1) g = 1;
    return (unsigned)std::min<size_t>(g, cap);
}

}  // namespace

void launch_pals_eval(const PalsConst& c, const double* params, double* mu, int32_t* flagS,
                      int32_t* flagP, cudaStream_t s) {
    const size_t N = (size_t)c.nx * c.ny * c.nz;
    pals_eval_kernel<<<grid_for(N, 256), 256, 5 * c.n_rbf * sizeof(double), s>>>(c, params, mu, flagS, flagP);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_mark_nodes(int32_t* flag, const int32_t* nodes, int n, cudaStream_t s) {
    if (n <= 0) return;
    mark_nodes_kernel<<<grid_for(n, 256), 256, 0, s>>>(flag, nodes, n);
    DOT_CUDA_TRY(cudaGetLastError());
}

size_t scan_temp_bytes(size_t n) { return ((n + kScanBlock - 1) / kScanBlock + 1) * sizeof(int32_t); }

void launch_exclusive_scan(const int32_t* in, int32_t* out, size_t n, int32_t* d_total, void* temp,
                           cudaStream_t s) {
    const int nb = (int)((n + kScanBlock - 1) / kScanBlock);
    int32_t* bsum = static_cast<int32_t*>(temp);
    scan_block_kernel<<<nb, kScanBlock, 0, s>>>(in, out, n, bsum);
    scan_sums_kernel<<<1, kScanBlock, 0, s>>>(bsum, nb, d_total);
    scan_add_kernel<<<nb, kScanBlock, 0, s>>>(out, n, bsum);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_compact(const int32_t* flag, const int32_t* pos, size_t n, int32_t* out_nodes, cudaStream_t s) {
    compact_kernel<<<grid_for(n, 256), 256, 0, s>>>(flag, pos, n, out_nodes);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_gather_rank(const int32_t* pos, const int32_t* nodes, int n, int32_t* out, cudaStream_t s) {
    if (n <= 0) return;
    gather_rank_kernel<<<grid_for(n, 256), 256, 0, s>>>(pos, nodes, n, out);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_pals_grad(const PalsConst& c, const double* params, const int32_t* S, int K, double* G,
                      cudaStream_t s) {
    if (K <= 0) return;
    pals_grad_kernel<<<grid_for(K, 128), 128, 5 * c.n_rbf * sizeof(double), s>>>(c, params, S, K, G);
    DOT_CUDA_TRY(cudaGetLastError());
}

void launch_sample_offsets(const int32_t* P, int nP, int nx, int ny, int nz, int TY, int ntiles,
                           int32_t* off, cudaStream_t s) {
    sample_offsets_kernel<<<grid_for((size_t)nz * ntiles + 1, 256), 256, 0, s>>>(P, nP, nx, ny, nz, TY, ntiles, off);
    DOT_CUDA_TRY(cudaGetLastError());
}

}  // namespace dot
