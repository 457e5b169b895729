// DMMA (mma.sync.m8n8k4.f64) throughput / latency probe on sm_100a: registers only, no
// memory traffic in the loop.  For W warps per CTA (one CTA per SM, 148 CTAs) and C
// independent accumulator chains per warp, prints achieved TFLOP/s.  Tells the
// contraction kernel how many warps x chains it needs to keep the FP64 tensor pipe busy.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

template <int C>
__global__ void probe(int iters, double* out) {
    double c[C][2];
    double a = threadIdx.x * 1e-3, b = blockIdx.x * 1e-3;
#pragma unroll
    for (int i = 0; i < C; ++i) c[i][0] = c[i][1] = 0.0;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int i = 0; i < C; ++i) dmma(c[i][0], c[i][1], a, b);
    }
    double s = 0;
#pragma unroll
    for (int i = 0; i < C; ++i) s += c[i][0] + c[i][1];
    if (s == 12345.0) out[0] = s;
}

template <int C>
void run(int warps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 4096;
    probe<C><<<sms, 32 * warps>>>(iters, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    probe<C><<<sms, 32 * warps>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 512.0 * C * iters * warps * (double)sms;
    printf("warps/SM %2d chains %2d : %.2f TFLOP/s  (%.1f clk per DMMA per SMSP at 1.965 GHz)\n", warps, C,
           fl / ms / 1e9, ms * 1e-3 * 1.965e9 / ((double)C * iters * warps / 4));
    cudaFree(out);
}

int main2();
int main() {
    main2();
    for (int w : {4, 8, 16}) {
        run<1>(w);
        run<2>(w);
        run<4>(w);
        run<8>(w);
        run<16>(w);
    }
    return 0;
}

// ---- inner loop of the segment contraction alone: per k4 1 U (LDS.128 + LDS.64) and 5 A
// (LDS.128 + LDS.64) fragments, 15 DMMA; shared tile static, no barriers.
template <int NQ>
__global__ void loop_probe(int iters, double* out) {
    extern __shared__ double2 sm2[];
    constexpr int RS = 20;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < 12 * 1024; i += blockDim.x) sm2[i] = make_double2(i * 1e-3, 1.0);
    __syncthreads();
    const double2* A = sm2 + ((warp >> 2) * 8 + (lane >> 2)) * RS;
    const double* As = reinterpret_cast<const double*>(sm2 + 4096) + ((warp >> 2) * 8 + (lane >> 2)) * RS;
    const double2* Ub = sm2 + 8192 + ((warp & 3) * 8 + (lane >> 2)) * RS;
    const double* Us = reinterpret_cast<const double*>(sm2 + 10240) + ((warp & 3) * 8 + (lane >> 2)) * RS;
    double p1[NQ][2] = {}, p2[NQ][2] = {}, p3[NQ][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int k4 = 0; k4 < 16; k4 += 4) {
            const int kk = k4 + (lane & 3) + (it & 1);
            const double2 u = Ub[kk];
            const double us = Us[kk];
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
                const double2 a = A[q * 32 * RS + kk];
                const double as = As[q * 32 * RS + kk];
                dmma(p1[q][0], p1[q][1], a.x, u.x);
                dmma(p2[q][0], p2[q][1], a.y, u.y);
                dmma(p3[q][0], p3[q][1], as, us);
            }
        }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < NQ; ++q) s += p1[q][0] + p2[q][1] + p3[q][0];
    if (s == 12345.0) out[0] = s;
}

template <int NQ>
void run_loop(int warps) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    const int iters = 2048;
    const size_t smem = 12 * 1024 * sizeof(double2);
    cudaFuncSetAttribute(loop_probe<NQ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    loop_probe<NQ><<<sms, 32 * warps, smem>>>(iters, out);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    loop_probe<NQ><<<sms, 32 * warps, smem>>>(iters, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fl = 512.0 * 3 * NQ * 4 * iters * warps * (double)sms;
    printf("loop NQ %d warps/SM %2d : %.2f TFLOP/s DMMA  (err %s)\n", NQ, warps, fl / ms / 1e9,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(out);
}

int main2() {
    for (int w : {4, 8, 12, 16}) {
        run_loop<5>(w);
        run_loop<2>(w);
    }
    return 0;
}
