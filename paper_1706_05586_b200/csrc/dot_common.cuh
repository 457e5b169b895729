// Shared device/host definitions of the B200 DOT library (internal).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <map>
#include <mutex>
#include <string>
#include <utility>
#include <vector>

#include "dot_b200.h"   // -I include

#define DOT_CUDA_TRY(expr)                                                            \
    do {                                                                              \
        cudaError_t _e = (expr);                                                      \
        if (_e != cudaSuccess) {                                                      \
            throw dot::Error(DOT_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
        }                                                                             \
    } while (0)

namespace dot {

struct Error {
    int code;
    std::string msg;
    Error(int c, std::string m) : code(c), msg(std::move(m)) {}
};

// Raise a kernel's dynamic shared-memory limit to at least `smem` on the current device.
// The attribute is per device, so the record of what was set is keyed by (kernel, device);
// thread-safe (problems may live on several devices / host threads of one process).
template <class K>
void ensure_smem(K kernel, size_t smem) {
    static std::mutex mtx;
    static std::map<std::pair<const void*, int>, size_t> done;
    int dev = 0;
    DOT_CUDA_TRY(cudaGetDevice(&dev));
    const auto key = std::make_pair(reinterpret_cast<const void*>(kernel), dev);
    std::lock_guard<std::mutex> lock(mtx);
    auto it = done.find(key);
    if (it != done.end() && it->second >= smem) return;
    DOT_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    done[key] = smem;
}

// ------------------------------------------------------------------ complex fp64
__host__ __device__ __forceinline__ double2 cmk(double re, double im) { return make_double2(re, im); }
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// a + b*c
__host__ __device__ __forceinline__ double2 cfma(double2 b, double2 c, double2 a) {
    return make_double2(fma(b.x, c.x, fma(-b.y, c.y, a.x)), fma(b.x, c.y, fma(b.y, c.x, a.y)));
}
__host__ __device__ __forceinline__ double2 cdiv(double2 a, double2 b) {
    // Smith's algorithm
    if (fabs(b.x) >= fabs(b.y)) {
        double r = b.y / b.x, d = b.x + b.y * r;
        return make_double2((a.x + a.y * r) / d, (a.y - a.x * r) / d);
    } else {
        double r = b.x / b.y, d = b.x * r + b.y;
        return make_double2((a.x * r + a.y) / d, (a.y * r - a.x) / d);
    }
}

// ------------------------------------------------------------- operator constants
// Row n of A(omega, p) (Eq. (2.1), R1-R3):
//   theta_k [ cx (2u - uW - uE) + cy (2u - uS - uN) + (mu + i shift) u ]
//   + cz (nzn_k u - uD - uU) + robin_k u,     shift = omega / nu
struct OpConst {
    int nx, ny, nz;
    double cx, cy, cz, robin;   // D/hx^2, D/hy^2, D/hz^2, 1/(2 hz)
    double dint;                // interior-plane diagonal without mu: 2 cx + 2 cy + 2 cz
};

__device__ __forceinline__ double theta_of(int k, int nz) { return (k == 0 || k == nz - 1) ? 0.5 : 1.0; }

// diagonal of A at plane k for absorption mu and shift
__device__ __forceinline__ double2 diag_of(const OpConst& c, int k, double mu, double shift) {
    double th = theta_of(k, c.nz);
    double nzn = (k == 0 || k == c.nz - 1) ? 1.0 : 2.0;
    double rob = (k == 0 || k == c.nz - 1) ? c.robin : 0.0;
    return make_double2(th * (2.0 * c.cx + 2.0 * c.cy + mu) + c.cz * nzn + rob, th * shift);
}

// Multi-shift CG state (cg_shift.cu).
constexpr int kMaxShift = 8;       // frequencies solved by one real seed
constexpr int kHist = 16;          // passes between folds of the shifted recurrences (history ring)
constexpr int kNumPartials = 8;    // per pair of seeds: rho(2) mu(2) nu(2) sigma_direct(2)

// Per-seed real CG state (double buffered by pass parity).
struct SeedState {
    double rho;                // rho_k = r_k^T r_k
    double alpha;              // alpha_k of the last active pass (a_{k-1} for the next one)
    double bnorm2;             // ||b~||_2^2
    int32_t done;              // 1 once converged / failed
    int32_t iters;             // iterations at convergence
    int32_t flag;              // 0 ok, DOT_ERR_NOCONV, DOT_ERR_BREAKDOWN
    int32_t pad;
};
// Per (seed, shift): zeta_{k-1}, zeta_k of the shifted residuals r_sigma = zeta r.
struct ShiftState {
    double2 zp, zc;
};
// Fold record of pass k for one (seed, shift): p_s <- zeta r_k + beta p_s; x_s += alpha p_s.
struct ShiftCoef {
    double2 zeta, beta, alpha;
    int32_t k;                 // pass the record belongs to (stale records are skipped)
    int32_t active;
};

}  // namespace dot
